"""Median layer latencies (CUDA events): decode layer-step (CUDA graph) and
prefill layer for Llama-3-8B on several partition sizes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.device.partition import DECODE, PREFILL
from paper_2504_19516_b200.workload import MODEL_PRESETS

cr = CoRunner(MODEL_PRESETS["llama3-8b"], 4096, 32, 2048)
out = {"pdl": os.environ.get("HP_PDL", "1")}
for sms in (148, 64, 32, 16, 8):
    out[f"decode_us_{sms}"] = 1e6 * cr.isolated(DECODE, sms, reps=9)
for sms in (148, 140):
    out[f"prefill_us_{sms}"] = 1e6 * cr.isolated(PREFILL, sms, reps=5)
print(json.dumps(out))
