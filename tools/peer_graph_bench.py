"""Fused TP all-reduce microbench: rank 0 of an emulated `world`-rank group (peers' flags pre-raised),
one linear replayed from a CUDA graph vs the plain gemm_swap.  args: world T N K sms [reps]"""
import sys

import torch
sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.peer import PeerAllReduce

dev = torch.device("cuda", 0)
world, T, N, K, sms = [int(a) for a in sys.argv[1:6]]
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 10
pr = PeerAllReduce.local_group(world, T, N, dev, device_epoch=True)[0]
pr.flags.fill_(2 ** 31 - 1)
x = torch.randn(T, K, device=dev).to(torch.bfloat16)
w = lib.tile_weight((torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16))
r = torch.randn(T, N, device=dev).to(torch.bfloat16)
out = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
import os
s = torch.cuda.Stream()
if os.environ.get("EAGER"):
    with torch.cuda.stream(s):
        for i in range(reps + 1):
            pr.linear(x, w, out, resid=r, max_ctas=sms)
            s.synchronize()
            print("eager call", i, pr.epoch_dev.tolist(), flush=True)
    sys.exit(0)
with torch.cuda.stream(s):
    pr.linear(x, w, out, resid=r, max_ctas=sms)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        pr.linear(x, w, out, resid=r, max_ctas=sms)
for i in range(reps):
    g.replay()
torch.cuda.synchronize()
print("ok", world, T, N, K, sms, pr.epoch_dev.tolist())

# timing: plain gemm_swap (RESID) vs the fused linear, both graph-replayed
ws, cnt = pr.workspace(K, sms)
y2 = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    lib.gemm_swap(x, w, y2, ws, cnt, lib.EPI_RESID, resid=r, max_ctas=sms)
    s.synchronize()
    with torch.cuda.graph(g2, stream=s):
        lib.gemm_swap(x, w, y2, ws, cnt, lib.EPI_RESID, resid=r, max_ctas=sms)
g3 = torch.cuda.CUDAGraph()  # GEMM half only
with torch.cuda.stream(s):
    with torch.cuda.graph(g3, stream=s):
        pr.gemm(x, w, 0, max_ctas=sms)
for name, gg in (("gemm_swap RESID", g2), ("fused linear", g), ("peer GEMM only", g3)):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        gg.replay()
    a.record()
    for _ in range(20):
        gg.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:18s} {a.elapsed_time(b) / 20 * 1e3:7.1f} us", flush=True)
