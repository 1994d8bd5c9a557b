"""Quick co-run exploration on the GPU (not the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.device.partition import DECODE, PREFILL
from paper_2504_19516_b200.workload import MODEL_PRESETS

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cr = CoRunner(MODEL_PRESETS["llama3-8b"], T, 32, 2048)
N = cr.n
print("N", N)
tp = {s: cr.isolated(PREFILL, s) for s in (148, 140, 132, 124, 116, 100, 84)}
print("prefill layer (us):", {k: round(v * 1e6, 1) for k, v in tp.items()})
td = {s: cr.isolated(DECODE, s) for s in (8, 16, 24, 32, 48, 64, 148)}
print("decode layer (us):", {k: round(v * 1e6, 1) for k, v in td.items()})
for dm in (8, 16, 24, 32, 48, 64):
    pm = N - dm
    n = max(1, round(tp.get(pm, tp[148]) / td[dm]))
    r = cr.corun(pm, dm, 4, n, time_upgate=True)
    ts = cr.time_sliced(4, n)
    print(f"dm={dm:3d} n={n:3d} corun {r.tokens_per_s/1e3:9.1f} ktok/s span {r.span_s*1e3:7.3f}ms "
          f"p50 prefill {r.p50(r.prefill_layer_s)*1e6:7.1f}us decode {r.p50(r.decode_layer_s)*1e6:6.1f}us "
          f"upgate {r.p50(r.upgate_s)*1e6:6.1f}us | time-sliced {ts.tokens_per_s/1e3:9.1f} ktok/s "
          f"span {ts.span_s*1e3:7.3f}ms speedup {ts.span_s/r.span_s:5.3f}", flush=True)
