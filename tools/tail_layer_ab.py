"""Stream-K tail A/B on whole prefill layers: Llama-3-8B layer at the
config-2 chunk sizes, (a) alone on pm SMs and (b) co-run beside the B=32
ctx-2048 decode graph on dm SMs (the bench's measurement), tail off/on
alternated A B A B A B to cancel clock drift.

    python tools/tail_layer_ab.py [T:pm:dm ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.device.partition import PREFILL, PartitionPool
from paper_2504_19516_b200.workload import MODEL_PRESETS

M = MODEL_PRESETS["llama3-8b"]
pool = PartitionPool(0)
points = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [
    (1024, 124, 24), (2048, 132, 16), (4096, 140, 8), (16384, 140, 8)]
weights = None
for T, pm, dm in points:
    cr = CoRunner(M, T, 32, 2048, pool=pool, weights=weights)
    weights = cr.layer.W
    res = {0: {"alone": [], "corun": [], "groups": []}, 1: {"alone": [], "corun": [], "groups": []}}
    for rep in range(3):
        for tail in (0, 1):
            lib.set_gemm_tail(tail)
            res[tail]["alone"].append(cr.isolated(PREFILL, pm, reps=5))
            r = cr.corun(pm, dm, 6, 1.4)
            res[tail]["corun"].append(statistics.median(r.prefill_layer_s))
    lib.set_gemm_tail(1)
    g1 = cr.corun(pm, dm, 4, 1.4, time_groups=True).group_s
    lib.set_gemm_tail(0)
    g0 = cr.corun(pm, dm, 4, 1.4, time_groups=True).group_s
    lib.set_gemm_tail(-1)
    row = {"T": T, "pm": pm, "dm": dm}
    for tail in (0, 1):
        k = "tail" if tail else "plain"
        row[f"{k}_alone_us"] = 1e6 * statistics.median(res[tail]["alone"])
        row[f"{k}_corun_us"] = 1e6 * statistics.median(res[tail]["corun"])
    row["groups_plain_us"] = {g: 1e6 * v for g, v in g0.items()}
    row["groups_tail_us"] = {g: 1e6 * v for g, v in g1.items()}
    row["corun_speedup"] = row["plain_corun_us"] / row["tail_corun_us"]
    print(json.dumps(row), flush=True)
