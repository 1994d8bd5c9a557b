"""Per-SM ingest of register-direct loads behind an L2 bulk prefetch
(hp_membw_pfldg) on green-context partitions, beside the plain LDG and
bulk-copy paths of tools/ldg_probe.py.

    python tools/pfldg_probe.py [sms ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.partition import DECODE, PartitionPool

pool = PartitionPool(0)
buf = torch.ones(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB
out = torch.zeros(4, device="cuda")
nbytes = buf.numel() * 4
so = lib.load()


def timed(st, fn, reps=4):
    ts = []
    with torch.cuda.stream(st.torch_stream):
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            a.record()
            fn()
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    return min(x.elapsed_time(y) for x, y in ts[1:]) * 1e-3


for sms in []:
    st = pool.phase(DECODE, sms)
    s = st.torch_stream.cuda_stream
    t = timed(st, lambda: lib.membw(buf, st.sms, 1, out, stream=st.torch_stream))
    print(f"sms {st.sms:3d} bulk {nbytes / t / 1e9 / st.sms:6.1f} GB/s/SM", flush=True)
    for threads in (256, 512, 1024):
        for U in (2, 4, 8):
            if threads * U * 2 * 4 > 65536 * 0.75:
                continue
            line = f"sms {st.sms:3d} pfldg T={threads:4d} U={U}:"
            for dist in (0, 2, 4, 8, 16, 32):
                t = timed(st, lambda: lib.check(so.hp_membw_pfldg(buf.data_ptr(), nbytes, st.sms, threads, U, dist,
                                                                  out.data_ptr(), s), "pfldg"))
                line += f"  d{dist} {nbytes / t / 1e9 / st.sms:6.1f}"
            print(line, flush=True)

# staged reader (bulk copy + multi-warp ld.shared read-back) vs register-direct
for sms in [int(a) for a in sys.argv[1:]] or [8, 16, 148]:
    st = pool.phase(DECODE, sms)
    s = st.torch_stream.cuda_stream
    for readers, ldgw, frac, rm in ((4, 0, 256, 0), (4, 0, 256, 1), (8, 0, 256, 1), (12, 0, 256, 1),
                                    (0, 8, 0, 1), (0, 16, 0, 1), (0, 19, 0, 1),
                                    (8, 8, 128, 1), (8, 8, 96, 1), (8, 11, 96, 1), (8, 11, 64, 1),
                                    (8, 11, 160, 1), (8, 11, 128, 0), (4, 12, 96, 1), (4, 12, 64, 1)):
        t = timed(st, lambda: lib.check(so.hp_membw_stage(buf.data_ptr(), nbytes, st.sms, readers, ldgw, frac, rm,
                                                          out.data_ptr(), s), "stage"))
        print(f"sms {st.sms:3d} stage readers={readers:2d} read={rm} ldg_warps={ldgw:2d} bulk={frac:3d}/256 "
              f"{nbytes / t / 1e9 / st.sms:6.1f} GB/s/SM", flush=True)
