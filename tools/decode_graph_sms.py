"""One-graph decode layer-step (Llama-3-8B, B tokens, ctx 2048) vs partition
size: median CUDA-event time of the graph replay per SM count.  Run once per
HP_SWAP_PAIR setting for the swap-GEMM pair/single A/B.

    HP_SWAP_PAIR=1 python tools/decode_graph_sms.py [B] [sms ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.device.partition import DECODE
from paper_2504_19516_b200.workload import MODEL_PRESETS

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sms = [int(a) for a in sys.argv[2:]] or [8, 16, 24, 32, 48, 64, 96, 148]
cr = CoRunner(MODEL_PRESETS["llama3-8b"], 1024, B, 2048)
out = {"B": B, "HP_SWAP_PAIR": os.environ.get("HP_SWAP_PAIR", "default")}
for n in sms:
    out[n] = round(1e6 * cr.isolated(DECODE, n, reps=7), 1)
print(json.dumps(out), flush=True)
