"""Per-kernel times of one Llama-3-8B decode layer-step (B=32, ctx 2048) on
green-context partitions: events between the launches (each kernel then
runs without its programmatic-launch overlap) beside the CUDA-graph replay
of the whole step, plus each kernel's algorithmic bytes and GB/s per SM.

    python tools/decode_breakdown.py [sms ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2504_19516_b200.device import lib
from paper_2504_19516_b200.device.corun import CoRunner
from paper_2504_19516_b200.device.layer import EPS
from paper_2504_19516_b200.device.partition import DECODE
from paper_2504_19516_b200.workload import MODEL_PRESETS

M = MODEL_PRESETS["llama3-8b"]
cr = CoRunner(M, 1024, 32, 2048)
L, sc, B = cr.layer, cr.dsc, cr.B
W = L.W
Hq, Hkv, d = L.Hq, L.Hkv, L.d
x, y = cr.dx, cr.dy
h = M.hidden
kv = 2 * 32 * 2048 * Hkv * d * 2 + 2 * 32 * Hkv * d * 2 + 2 * 32 * h * 2
steps = [
    ("rmsnorm1", 4 * B * h, lambda s, st: lib.rmsnorm(x, W.attn_norm, sc.xn[:B], EPS, s, st)),
    ("qkv", W.w_qkv.numel() * 2, lambda s, st: lib.gemm_swap(sc.xn[:B], W.w_qkv, sc.qkv[:B], sc.gemm_ws, sc.gemm_cnt,
                                                            lib.EPI_STORE, max_ctas=s, stream=st)),
    ("rope_kv", 4 * B * (Hq + 2 * Hkv) * d, lambda s, st: lib.rope_kv_write(sc.qkv[:B], Hq, Hkv, d, cr.d_pos, L.rope,
                                                                           cr.d_slots, cr.dcache.k, cr.dcache.v,
                                                                           cr.dcache.page, max_ctas=s, stream=st)),
    ("attn", kv, lambda s, st: lib.decode_attn(sc.qkv[:B], cr.dcache.k, cr.dcache.v, cr.block_table, cr.ctx,
                                               sc.attn[:B], Hq, Hkv, d, cr.dcache.page, L.scale, ws=sc.attn_ws,
                                               max_ctas=s, stream=st)),
    ("o_proj", W.w_o.numel() * 2, lambda s, st: lib.gemm_swap(sc.attn[:B], W.w_o, sc.h[:B], sc.gemm_ws, sc.gemm_cnt,
                                                             lib.EPI_RESID, resid=x, max_ctas=s, stream=st)),
    ("rmsnorm2", 4 * B * h, lambda s, st: lib.rmsnorm(sc.h[:B], W.mlp_norm, sc.xn[:B], EPS, s, st)),
    ("mlp_up_gate", W.w_ug.numel() * 2, lambda s, st: lib.gemm_swap(sc.xn[:B], W.w_ug, sc.act[:B], sc.gemm_ws,
                                                                   sc.gemm_cnt, lib.EPI_SILU, max_ctas=s, stream=st)),
    ("mlp_down", W.w_down.numel() * 2, lambda s, st: lib.gemm_swap(sc.act[:B], W.w_down, y, sc.gemm_ws, sc.gemm_cnt,
                                                                  lib.EPI_RESID, resid=sc.h[:B], max_ctas=s,
                                                                  stream=st)),
]
for sms in [int(a) for a in sys.argv[1:]] or [8, 16, 32, 148]:
    st = cr.pool.phase(DECODE, sms)
    ts = {name: [] for name, _, _ in steps}
    with torch.cuda.stream(st.torch_stream):
        for rep in range(6):
            lib.hold(st.torch_stream, 100_000)
            evs = []
            for name, _, fn in steps:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn(st.sms, st.torch_stream)
                b.record()
                evs.append((name, a, b))
            torch.cuda.synchronize()
            if rep:
                for name, a, b in evs:
                    ts[name].append(a.elapsed_time(b) * 1e3)
    graph_us = 1e6 * cr.isolated(DECODE, sms, reps=7)
    out = {"sms": st.sms, "graph_step_us": graph_us}
    tot = 0.0
    for name, nbytes, _ in steps:
        us = statistics.median(ts[name])
        tot += us
        out[name] = {"us": round(us, 1), "GBps_per_SM": round(nbytes / us / 1e3 / st.sms, 1)}
    out["sum_kernels_us"] = tot
    print(json.dumps(out), flush=True)
