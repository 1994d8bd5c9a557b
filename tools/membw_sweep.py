"""HBM bandwidth vs SM count (green-context partitions), both access paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool

pool = PartitionPool(0)
N = pool.n
buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB
out = torch.zeros(4, device="cuda")
nbytes = buf.numel() * 4
for method in (0, 1):
    for sms in [8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 144, N]:
        st = pool.phase(DECODE, sms)
        ctas = st.sms * (4 if method == 0 else 1)
        ts = []
        with torch.cuda.stream(st.torch_stream):
            for i in range(4):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda._sleep(100000)
                a.record()
                lib.membw(buf, ctas, method, out, stream=st.torch_stream)
                b.record()
                ts.append((a, b))
        torch.cuda.synchronize()
        t = min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3
        print(f"method {method} sms {st.sms:3d}: {nbytes / t / 1e9:8.1f} GB/s  ({nbytes / t / 1e9 / st.sms:6.1f} GB/s/SM)", flush=True)
