import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
if len(sys.argv) > 1:
    lib.load(sys.argv[1])
from paper_2504_19516_b200.device import kbench
res = []
for sms in (148, 32):
    kbench.bench_gemm_swap(32, 6144, 4096, 0, sms, res)
    kbench.bench_gemm_swap(32, 28672, 4096, 2, sms, res)
    kbench.bench_decode_attn(32, 2048, 32, 8, sms, res)
kbench.bench_gemm(4096, 28672, 4096, 2, 148, res)
kbench.bench_prefill_attn(4096, 32, 8, 148, res)
