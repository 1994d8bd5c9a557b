"""Prefill GEMM time at tile width 128 vs 256 (HP_GEMM_BN set by the caller)
for the Llama-3-8B layer shapes and several grid sizes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.kbench import timeit
DEV = torch.device("cuda", 0)
res = {}
shapes = [("qkv", 6144, 4096, lib.EPI_STORE), ("o", 4096, 4096, lib.EPI_RESID),
          ("ug", 28672, 4096, lib.EPI_SILU), ("down", 4096, 14336, lib.EPI_RESID)]
for T in (1024, 2048, 4096):
    for name, N, K, epi in shapes:
        x = torch.randn(T, K, device=DEV).to(torch.bfloat16)
        w = lib.tile_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
        on = N // 2 if epi == lib.EPI_SILU else N
        y = torch.empty(T, on, device=DEV, dtype=torch.bfloat16)
        r = torch.randn(T, on, device=DEV).to(torch.bfloat16) if epi == lib.EPI_RESID else None
        for sms in (148, 140, 132, 116):
            t = timeit(lambda: lib.gemm(x, w, y, epi, resid=r, max_ctas=sms), iters=8)
            res[f"{name}/{T}/{sms}"] = round(t * 1e6, 1)
print(os.environ.get("HP_GEMM_BN", "auto"), json.dumps(res))
