import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device import lib
if len(sys.argv) > 1:
    lib.load(sys.argv[1])
from paper_2504_19516_b200.device import kbench
res = []
for sms in (32, 148):
    kbench.bench_gemm_swap(32, 6144, 4096, 0, sms, res)
    kbench.bench_gemm_swap(32, 28672, 4096, 2, sms, res)
