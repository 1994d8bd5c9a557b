import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib, kbench
res = []
for sms in (32, 148):
    for T in (32, 64, 128, 256):
        kbench.bench_gemm_swap(T, 6144, 4096, 0, sms, res)
    for T in (32, 128):
        kbench.bench_gemm(T, 6144, 4096, 0, sms, res)
        kbench.bench_gemm(T, 28672, 4096, 2, sms, res)
for r in res:
    if r["kernel"] == "gemm":
        N, K = r["N"], r["K"]
        print("gemm T", r["T"], "N", N, "sms", r["sms"], "GB/s weights", N * K * 2 / (r["us"] * 1e-6) / 1e9)
