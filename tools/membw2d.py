"""1-D bulk vs 2-D TMA box streaming at several SM counts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool

pool = PartitionPool(0)
rows, cols = 131072, 4096  # 1 GiB bf16
buf = torch.ones(rows, cols, dtype=torch.bfloat16, device="cuda")
out = torch.zeros(4, device="cuda")
nbytes = rows * cols * 2


def run(fn, st):
    ts = []
    with torch.cuda.stream(st.torch_stream):
        for i in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    return min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3


for sms in (8, 32, 64, 148):
    st = pool.phase(DECODE, sms)
    t1 = run(lambda: lib.load().hp_membw(buf.data_ptr(), nbytes, st.sms, 1, out.data_ptr(), st.stream), st)
    line = f"sms {st.sms:3d}: bulk1d {nbytes/t1/1e9:7.1f} GB/s"
    for br in (32, 64, 128, 256):
        t = run(lambda: lib.check(lib.load().hp_membw2d(buf.data_ptr(), rows, cols, br, st.sms, out.data_ptr(), st.stream)), st)
        line += f" | 2d box{br:3d} {nbytes/t/1e9:7.1f}"
    # 2-D boxes over a narrow matrix (row pitch 128 B: contiguous boxes)
    t = run(lambda: lib.check(lib.load().hp_membw2d(buf.data_ptr(), rows * cols // 64, 64, 128, st.sms, out.data_ptr(), st.stream)), st)
    line += f" | 2d box128 contiguous {nbytes/t/1e9:7.1f}"
    print(line, flush=True)
