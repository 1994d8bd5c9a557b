"""Decode (swap-AB stream-K) GEMM GB/s of weights when confined to `sms`
CTAs, llama3-8b decode batch 32 shapes, L2 flushed.   python tools/swap_sms.py [sms ...]
SW_GREEN=1: inside a green context of `sms` SMs (the co-run's condition: both
SMs of a TPC busy) instead of `sms` CTAs on an otherwise idle GPU."""
import contextlib
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
T = 32
shapes = [("qkv", 6144, 4096, lib.EPI_STORE), ("o_proj", 4096, 4096, lib.EPI_RESID),
          ("up_gate", 28672, 4096, lib.EPI_SILU), ("down", 4096, 14336, lib.EPI_RESID)]
pool = None
if os.environ.get("SW_GREEN"):
    from paper_2504_19516_b200.device.partition import DECODE, PartitionPool
    pool = PartitionPool(0)
for sms in [int(a) for a in sys.argv[1:]] or [8, 16, 148]:
    ctx = torch.cuda.stream(pool.phase(DECODE, sms).torch_stream) if pool else contextlib.nullcontext()
    ctx.__enter__()
    tot_b, tot_t = 0, 0.0
    for name, N, K, epi in shapes:
        x = torch.randn(T, K, device=dev).to(torch.bfloat16)
        w = lib.tile_weight((torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16))
        r = torch.randn(T, N, device=dev).to(torch.bfloat16)
        y = torch.empty(T, N // 2 if epi == lib.EPI_SILU else N, device=dev, dtype=torch.bfloat16)
        ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, sms) // 4 + 1, device=dev)
        cnt = torch.zeros(N // 128 * 8, device=dev, dtype=torch.int32)
        ts = []
        for i in range(6):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lib.gemm_swap(x, w, y, ws, cnt, epi, resid=r if epi == lib.EPI_RESID else None, max_ctas=sms,
                          stream=torch.cuda.current_stream())
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        nb = N * K * 2
        tot_b += nb
        tot_t += t
        print(f"sms {sms:4d} {name:8s} {t * 1e6:8.1f} us {nb / t / 1e9:7.1f} GB/s {nb / t / 1e9 / sms:6.1f} GB/s/SM",
              flush=True)
    print(f"sms {sms:4d} all      {tot_t * 1e6:8.1f} us {tot_b / tot_t / 1e9:7.1f} GB/s {tot_b / tot_t / 1e9 / sms:6.1f} GB/s/SM")
    ctx.__exit__(None, None, None)
