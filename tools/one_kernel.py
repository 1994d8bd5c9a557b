"""Run a single hot-path kernel a few times (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import sys

import torch

from paper_2504_19516_b200.device import lib

DEV = torch.device("cuda", 0)
which = sys.argv[1]
sms = int(sys.argv[2]) if len(sys.argv) > 2 else 148
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if which.startswith("swap"):
    T, N, K = 32, 4096, 4096
    if which == "swap_qkv":
        N = 6144
    epi = lib.EPI_STORE
    if which == "swap_ug":  # mlp_up_gate, the largest decode GEMM (235 MB of weights)
        N, epi = 28672, lib.EPI_SILU
    x = torch.randn(T, K, device=DEV).to(torch.bfloat16)
    w = lib.tile_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
    y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, sms) // 4, device=DEV)
    cnt = torch.zeros(N // 128, device=DEV, dtype=torch.int32)
    for _ in range(reps):
        lib.gemm_swap(x, w, y, ws, cnt, epi, max_ctas=sms)
elif which == "decode_attn":
    B, ctx, Hq, Hkv, d, page = 32, 2048, 32, 8, 128, 64
    pages = ctx // page
    kc = torch.randn(B * pages, Hkv, page, d, device=DEV).to(torch.bfloat16)
    vc = torch.randn_like(kc)
    bt = torch.randperm(B * pages, device=DEV).to(torch.int32).view(B, pages)
    q = torch.randn(B, Hq * d, device=DEV).to(torch.bfloat16)
    out = torch.empty_like(q)
    cl = torch.full((B,), ctx, device=DEV, dtype=torch.int32)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 512) // 4, device=DEV)
    for _ in range(reps):
        lib.decode_attn(q, kc, vc, bt, cl, out, Hq, Hkv, d, page, 1 / math.sqrt(d), ws=ws, max_ctas=sms)
elif which.startswith("gemm"):
    T = int(which[4:] or 4096)
    x = torch.randn(T, 4096, device=DEV).to(torch.bfloat16)
    w = lib.tile_weight((torch.randn(28672, 4096, device=DEV) * 0.02).to(torch.bfloat16))
    y = torch.empty(T, 14336, device=DEV, dtype=torch.bfloat16)
    for _ in range(reps):
        lib.gemm(x, w, y, lib.EPI_SILU, max_ctas=sms)
elif which.startswith("attn"):
    T = int(which[4:] or 4096)
    Hq, Hkv, d = 32, 8, 128
    qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=DEV).to(torch.bfloat16)
    q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    cu = torch.tensor([0, T], device=DEV, dtype=torch.int32)
    for _ in range(reps):
        lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms)
torch.cuda.synchronize()
print("done", which)
