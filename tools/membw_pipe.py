import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool
pool = PartitionPool(0)
buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
out = torch.zeros(4, device="cuda")
nbytes = buf.numel() * 4
def bw(st, fn):
    ts = []
    with torch.cuda.stream(st.torch_stream):
        for i in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    t = min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3
    return nbytes / t / 1e9 / st.sms
st = pool.phase(DECODE, 32)
for np_ in (1, 2, 4, 8):
    line = f"sms 32 pipe producers {np_}:"
    for kb in (16, 32):
        if 192 // kb < np_:
            continue
        v = bw(st, lambda: lib.check(lib.load().hp_membw_pipe(buf.data_ptr(), nbytes, st.sms, kb, np_, out.data_ptr(), st.stream)))
        line += f"  {kb}KB {v:6.1f}"
    print(line, flush=True)
