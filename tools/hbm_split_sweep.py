"""Dual-roofline co-run sweep: prefill layer (T tokens) on N - dm SMs with
per-GEMM events while the dm side streams decode attention (B=32, ctx
2048); prints attention GB/s (co-run and alone) and the GEMMs' fraction of
the partition's burst peak.

    python tools/hbm_split_sweep.py T dm [dm ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import _peaks, hbm_targets  # noqa: E402
from paper_2504_19516_b200.device.corun import CoRunner  # noqa: E402
from paper_2504_19516_b200.device.layer import LayerWeights  # noqa: E402
from paper_2504_19516_b200.workload import MODEL_PRESETS  # noqa: E402

m = MODEL_PRESETS["llama3-8b"]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
T = int(sys.argv[1])
cr = CoRunner(m, T, 32, 2048, weights=LayerWeights.random_device(m, dev, g))
hbm, tf, _, _ = _peaks()
for dm in [int(a) for a in sys.argv[2:]]:
    r = hbm_targets(cr, dm, hbm, tf)
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if k != "note"}),
          flush=True)
