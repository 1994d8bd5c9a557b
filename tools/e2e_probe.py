"""Where does the end-to-end (pinned host I/O) co-run lose time?  Runs
CoRunner.corun_e2e variants at the bench's headline split and prints
layer-tokens/s for each (device-timed, CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device.corun import CoRunner  # noqa: E402
from paper_2504_19516_b200.device.layer import LayerWeights  # noqa: E402
from paper_2504_19516_b200.workload import MODEL_PRESETS  # noqa: E402

m = MODEL_PRESETS["llama3-8b"]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cr = CoRunner(m, T, 32, 2048, weights=LayerWeights.random_device(m, dev, g))
pm, dm, r, K = 140, 8, 1.45, 30
h = m.hidden
pin = [torch.empty(n, h, dtype=torch.bfloat16, pin_memory=True) for n in (T, T, 32, 32)]
out = {}
for _ in range(2):
    out["device_only"] = cr.corun(pm, dm, K, r).tokens_per_s
    for chunks in (1, 4):
        cr.e2e_chunks = chunks
        out[f"e2e_chunks{chunks}"] = cr.corun_e2e(pm, dm, K, r, *pin).tokens_per_s
    cr.e2e_chunks = 1
    cr.e2e_decode_io = False
    out["e2e_no_decode_io"] = cr.corun_e2e(pm, dm, K, r, *pin).tokens_per_s
    cr.e2e_decode_io = True
    cr.e2e_prefill_io = False
    out["e2e_no_prefill_io"] = cr.corun_e2e(pm, dm, K, r, *pin).tokens_per_s
    cr.e2e_prefill_io = True
print(json.dumps({k: round(v / 1e6, 3) for k, v in out.items()}))
