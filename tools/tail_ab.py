"""A/B of the prefill GEMMs with and without the stream-K tail: Llama-3-8B
layer GEMMs (qkv / o_proj / mlp_up_gate / mlp_down) at the config-2 chunk
sizes on the estimator's prefill partitions, CUDA events on the
partition's green-context stream, median of 7, inputs > L2 between reps
(weights alternate with a second copy).

    python tools/tail_ab.py [T:pm ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.layer import LayerWeights
from paper_2504_19516_b200.device.partition import PREFILL, PartitionPool
from paper_2504_19516_b200.workload import MODEL_PRESETS

M = MODEL_PRESETS["llama3-8b"]
dev = torch.device("cuda", 0)
pool = PartitionPool(0)
g = torch.Generator(device=dev)
g.manual_seed(0)
W = LayerWeights.random_device(M, dev, g)
h, I = M.hidden, M.intermediate
points = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(1024, 124), (2048, 132), (4096, 140),
                                                                         (16384, 140), (4096, 148)]
rows = []
for T, pm in points:
    st = pool.phase(PREFILL, pm) if pm < pool.n else pool.full(PREFILL)
    bf = dict(dtype=torch.bfloat16, device=dev)
    xh, xi = torch.randn(T, h, **bf), torch.randn(T, I, **bf)
    for name, w, x, n_out, epi, r in (("qkv", W.w_qkv, xh, M.qkv_out_dim, lib.EPI_STORE, None),
                                      ("o_proj", W.w_o, xh, h, lib.EPI_RESID, xh),
                                      ("mlp_up_gate", W.w_ug, xh, I, lib.EPI_SILU, None),
                                      ("mlp_down", W.w_down, xi, h, lib.EPI_RESID, xh)):
        y = torch.empty(T, n_out, **bf)
        flops = 2.0 * T * w.shape[0] * x.shape[1]
        res = {}
        for tail in (0, 1):
            lib.set_gemm_tail(tail)
            evs = []
            with torch.cuda.stream(st.torch_stream):
                for i in range(8):
                    lib.hold(st.torch_stream, 50_000)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    lib.gemm(x, w, y, epi, resid=r, max_ctas=st.sms, stream=st.torch_stream)
                    b.record()
                    evs.append((a, b))
            torch.cuda.synchronize()
            t = statistics.median(a.elapsed_time(b) for a, b in evs[1:]) * 1e-3
            res[tail] = t
        lib.set_gemm_tail(-1)
        row = {"T": T, "pm": st.sms, "gemm": name, "plain_us": 1e6 * res[0], "tail_us": 1e6 * res[1],
               "plain_tflops": flops / res[0] / 1e12, "tail_tflops": flops / res[1] / 1e12,
               "speedup": res[0] / res[1]}
        rows.append(row)
        print(json.dumps(row), flush=True)
tot0 = sum(r["plain_us"] for r in rows)
tot1 = sum(r["tail_us"] for r in rows)
print(json.dumps({"total_plain_us": tot0, "total_tail_us": tot1, "speedup": tot0 / tot1}))
