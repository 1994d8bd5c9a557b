"""Prefill attention TFLOP/s (k_fa2) at the bench shapes; HP_LIB=<path>
loads an alternative libb200hot.so for A/B comparisons.
    python tools/fa_ab.py"""
import os
import sys

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

if os.environ.get("HP_LIB"):
    lib.load(os.environ["HP_LIB"])
from paper_2504_19516_b200.device import kbench  # noqa: E402

res = []
for T, sms in ((4096, 148), (4096, 140), (16384, 148), (1024, 148)):
    kbench.bench_prefill_attn(T, 32, 8, sms, res)
for r in res:
    print(r, flush=True)
