"""Decode swap-AB GEMM time vs grid size on the full GPU (T = 32, Llama-3-8B
layer shapes), back-to-back launches between two events (the graph's
steady state, PDL prologue overlap included).

    python tools/swap_ctas.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

dev = torch.device("cuda", 0)
T = 32
res = {}
for name, N, K, epi in (("qkv", 6144, 4096, lib.EPI_STORE), ("o_proj", 4096, 4096, lib.EPI_RESID),
                        ("up_gate", 28672, 4096, lib.EPI_SILU), ("down", 4096, 14336, lib.EPI_RESID)):
    x = torch.randn(T, K, device=dev).to(torch.bfloat16)
    w = lib.tile_weight((torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16))
    y = torch.empty(T, N // 2 if epi == lib.EPI_SILU else N, device=dev, dtype=torch.bfloat16)
    r = torch.randn(T, N, device=dev).to(torch.bfloat16) if epi == lib.EPI_RESID else None
    ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, 148) // 4 + 1, device=dev)
    cnt = torch.zeros(N // 128 * 8, device=dev, dtype=torch.int32)
    row = {}
    for ctas in [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else "16,32,48,64,80,96,112,128,148".split(","))]:
        def go():
            lib.gemm_swap(x, w, y, ws, cnt, epi, resid=r, max_ctas=ctas)
        go()
        ts = []
        for _ in range(7):
            torch.cuda._sleep(100_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                go()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / 20)
        row[ctas] = round(sorted(ts)[3], 2)
    res[name] = {"MB": N * K * 2 / 1e6, "us_by_ctas": row}
    print(name, json.dumps(res[name]), flush=True)
