"""Diagnose stream-K tail vs plain rounds on one GEMM shape."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

T, N, K, ctas = (int(a) for a in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 6144, 4096, 140)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
x = (torch.randn(T, K, generator=g, device=dev)).to(torch.bfloat16)
w = (torch.randn(N, K, generator=g, device=dev) * 0.05).to(torch.bfloat16)
wt = lib.tile_weight(w)
ys = {}
for tail in (0, 1):
    lib.set_gemm_tail(tail)
    y = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
    lib.gemm(x, wt, y, lib.EPI_STORE, max_ctas=ctas)
    torch.cuda.synchronize()
    ys[tail] = y.float()
ref = x.float() @ w.float().T
e0 = (ys[0] - ref).abs()
e1 = (ys[1] - ref).abs()
d = (ys[1] - ys[0]).abs()
ulp = torch.pow(2.0, torch.floor(torch.log2(ys[0].abs().clamp_min(1e-30))) - 7)
print("max err plain", e0.max().item(), "tail", e1.max().item())
print("differing elements", int((d > 0).sum()), "of", d.numel())
print("max d/ulp", (d / ulp).max().item())
idx = torch.nonzero(d / ulp > 1.5)
print("elements > 1.5 ulp:", idx.shape[0])
for r, c in idx[:10].tolist():
    print(r, c, "plain", ys[0][r, c].item(), "tail", ys[1][r, c].item(), "ref", ref[r, c].item())
if idx.shape[0]:
    rows = idx[:, 0] // 256
    cols = idx[:, 1] // 256
    tiles = sorted(set(zip(rows.tolist(), cols.tolist())))
    print("bad (m,n) tiles:", tiles[:40], len(tiles))
