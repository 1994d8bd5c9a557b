"""What slows the prefill layer in the co-run: the T=4096 Llama-3-8B prefill
layer on 140 SMs timed (CUDA events, median of 6 layers) while the 8-SM side
runs (a) nothing, (b) legacy-MMA spin (SM power, no memory traffic),
(c) a bulk-copy HBM stream (memory traffic, no math), (d) the decode graph.

    python tools/corun_interference.py [T pm dm]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.workload import MODEL_PRESETS

T, pm, dm = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 140, 8)
cr = CoRunner(MODEL_PRESETS["llama3-8b"], T, 32, 2048)
ps, ds = cr.pool.split(pm, dm)
g = cr.decode_graph(ds)
so = lib.load()
buf = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
out = torch.zeros(4, device="cuda")
cyc = torch.zeros(256, dtype=torch.int64, device="cuda")
res = {}
for mode in ("idle", "mma_spin", "hbm_stream", "decode_graph", "idle"):
    layers = 6
    with torch.cuda.stream(ps.torch_stream):
        cr.prefill_layer(ps)
    torch.cuda.synchronize()
    ctrl = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(ctrl)
    ps.torch_stream.wait_event(start)
    ds.torch_stream.wait_event(start)
    with torch.cuda.stream(ds.torch_stream):
        if mode == "mma_spin":
            lib.check(so.hp_hmma_rate(400000, 8, ds.sms, 512, cyc.data_ptr(), ds.stream), "hmma")
        elif mode == "hbm_stream":
            for _ in range(20):
                lib.membw(buf, ds.sms, 1, out, stream=ds.torch_stream)
        elif mode == "decode_graph":
            for _ in range(12):
                g.replay()
    evs = []
    with torch.cuda.stream(ps.torch_stream):
        for _ in range(layers):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ps.torch_stream)
            cr.prefill_layer(ps)
            b.record(ps.torch_stream)
            evs.append((a, b))
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1e3 for a, b in evs]
    res.setdefault(mode, []).append(round(statistics.median(ts[1:-1]), 1))
print(json.dumps({"T": T, "pm": pm, "dm": dm, "prefill_layer_us": res}))
