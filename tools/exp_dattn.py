"""Decode attention / decode GEMM bandwidth vs SM count (Llama-3-8B, B=32, ctx 2048).
usage: python tools/exp_dattn.py [lib.so] [--gemm]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_19516_b200.device import lib
args = [a for a in sys.argv[1:] if not a.startswith("--")]
if args:
    lib.load(args[0])
    print("lib", args[0])
from paper_2504_19516_b200.device import kbench
res = []
for sms in (8, 16, 32, 64, 148):
    kbench.bench_decode_attn(32, 2048, 32, 8, sms, res)
if "--gemm" in sys.argv:
    for sms in (8, 16, 32):
        kbench.bench_gemm_swap(32, 28672, 4096, 2, sms, res)
        kbench.bench_gemm_swap(32, 4096, 14336, 1, sms, res)
