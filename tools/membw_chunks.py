"""Per-SM bulk-copy throughput vs chunk size (single issuing thread, 192 KB in flight)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool

pool = PartitionPool(0)
buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
out = torch.zeros(4, device="cuda")
nbytes = buf.numel() * 4
for sms in (8, 32, 148):
    st = pool.phase(DECODE, sms)
    line = f"sms {st.sms:3d}:"
    for m in (10, 11, 12, 13, 14):
        ts = []
        with torch.cuda.stream(st.torch_stream):
            for i in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(100000)
                a.record()
                lib.membw(buf, st.sms, m, out, stream=st.torch_stream)
                b.record()
                ts.append((a, b))
        torch.cuda.synchronize()
        t = min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3
        line += f"  {4 << (m - 10):2d}KB {nbytes / t / 1e9 / st.sms:6.1f} GB/s/SM"
    print(line, flush=True)
