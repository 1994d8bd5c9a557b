import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool
pool = PartitionPool(0)
buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
out = torch.zeros(4, device="cuda")
nbytes = buf.numel() * 4
def bw(st, method):
    ts = []
    with torch.cuda.stream(st.torch_stream):
        for i in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            a.record()
            lib.membw(buf, st.sms, method, out, stream=st.torch_stream)
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    t = min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3
    return nbytes / t / 1e9 / st.sms
st = pool.phase(DECODE, 32)
for blocked in (0, 1):
    for wl in (0, 2):
        line = f"sms 32 blocked {blocked} warps {1 << wl}:"
        for k in (2, 3):
            line += f"  {4 << k:2d}KB {bw(st, 10 + k + 8 * wl + 1024 * blocked):6.1f}"
        print(line, flush=True)
