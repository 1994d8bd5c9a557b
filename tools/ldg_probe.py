"""Per-SM streaming bandwidth of register-direct loads vs the bulk-copy path,
on green-context partitions of `sms` SMs, and the legacy mma.sync rate.

    python tools/ldg_probe.py [sms ...]

Lines: `ldg T=<threads/CTA> c=<CTAs/SM> U=<unroll> na=<0|1>` (hp_membw_ldg),
`bulk` (hp_membw method 1: TMA 1-D bulk copies into a 6 x 32 KB ring),
`hmma warps=<w> chains=<c>` (MAC/clk/SM of mma.sync.m16n8k16).
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


# mma.sync rate, one CTA on one SM
cyc = torch.zeros(4, dtype=torch.int64, device="cuda")
for warps in (4, 8, 16):
    for chains in (1, 2, 4, 8):
        n = 4096
        lib.check(so.hp_hmma_rate(n, chains, 1, warps * 32, cyc.data_ptr(), 0), "hmma")
        torch.cuda.synchronize()
        c = int(cyc[0].item())
        macs = warps * n * chains * 16 * 8 * 16
        print(f"hmma warps={warps:2d} chains={chains}: {macs / c:7.1f} MAC/clk/SM", flush=True)

sms_list = [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64, 148]
for sms in sms_list:
    st = pool.phase(DECODE, sms)
    s = st.torch_stream.cuda_stream
    for lw in (4, 8, 16):
        for frac in (256, 192, 160, 128, 96, 0, 1024 + 256, 1024 + 192, 1024 + 160, 1024 + 128, 1024 + 96):
            t = timed(st, lambda: lib.check(so.hp_membw_mix(buf.data_ptr(), nbytes, st.sms, lw, frac,
                                                            out.data_ptr(), s), "mix"))
            print(f"sms {st.sms:3d} mix ldg_warps={lw:2d} bulk={frac % 1024:3d}/256 read={frac // 1024} "
                  f"{nbytes / t / 1e9:8.1f} GB/s {nbytes / t / 1e9 / st.sms:6.1f} /SM", flush=True)
for sms in sms_list:
    st = pool.phase(DECODE, sms)
    s = st.torch_stream.cuda_stream
    t = timed(st, lambda: lib.membw(buf, st.sms, 1, out, stream=st.torch_stream))
    print(f"sms {st.sms:3d} bulk               {nbytes / t / 1e9:8.1f} GB/s {nbytes / t / 1e9 / st.sms:6.1f} /SM",
          flush=True)
    for threads, cps in ((256, 1), (512, 1), (1024, 1), (512, 2), (256, 4)):
        for U in (4, 8, 16):
            if threads * cps * U * 2 * 4 > 65536 * 0.75:  # data registers would not fit
                continue
            for na in (1,):
                try:
                    t = timed(st, lambda: lib.check(so.hp_membw_ldg(buf.data_ptr(), nbytes, st.sms * cps, threads, U,
                                                                na, out.data_ptr(), s), "ldg"))
                except Exception as e:  # noqa: BLE001
                    print(f"sms {st.sms:3d} ldg T={threads} c={cps} U={U}: {e}", flush=True)
                    continue
                print(f"sms {st.sms:3d} ldg T={threads:4d} c={cps} U={U:2d} na={na} "
                      f"{nbytes / t / 1e9:8.1f} GB/s {nbytes / t / 1e9 / st.sms:6.1f} /SM", flush=True)
