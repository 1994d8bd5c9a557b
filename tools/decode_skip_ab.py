"""What the small decode kernels cost inside the one-graph decode step:
graph replay of the full Llama-3-8B decode layer-step (B=32, ctx 2048) vs the
same graph without the two RMSNorms and/or the RoPE + KV-write launch
(numerically wrong, timing only), on green-context partitions.

    python tools/decode_skip_ab.py [sms ...]
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


def step(s, st, norms=True, rope=True):
    if norms:
        lib.rmsnorm(x, W.attn_norm, sc.xn[:B], EPS, s, st)
    lib.gemm_swap(sc.xn[:B], W.w_qkv, sc.qkv[:B], sc.gemm_ws, sc.gemm_cnt, lib.EPI_STORE, max_ctas=s, stream=st)
    if rope:
        lib.rope_kv_write(sc.qkv[:B], Hq, Hkv, d, cr.d_pos, L.rope, cr.d_slots, cr.dcache.k, cr.dcache.v,
                          cr.dcache.page, max_ctas=s, stream=st)
    lib.decode_attn(sc.qkv[:B], cr.dcache.k, cr.dcache.v, cr.block_table, cr.ctx, sc.attn[:B], Hq, Hkv, d,
                    cr.dcache.page, L.scale, ws=sc.attn_ws, max_ctas=s, stream=st)
    lib.gemm_swap(sc.attn[:B], W.w_o, sc.h[:B], sc.gemm_ws, sc.gemm_cnt, lib.EPI_RESID, resid=x, max_ctas=s,
                  stream=st)
    if norms:
        lib.rmsnorm(sc.h[:B], W.mlp_norm, sc.xn[:B], EPS, s, st)
    lib.gemm_swap(sc.xn[:B], W.w_ug, sc.act[:B], sc.gemm_ws, sc.gemm_cnt, lib.EPI_SILU, max_ctas=s, stream=st)
    lib.gemm_swap(sc.act[:B], W.w_down, y, sc.gemm_ws, sc.gemm_cnt, lib.EPI_RESID, resid=sc.h[:B], max_ctas=s,
                  stream=st)


for sms in [int(a) for a in sys.argv[1:]] or [8, 32, 148]:
    st = cr.pool.phase(DECODE, sms)
    out = {"sms": st.sms}
    for name, kw in (("full", {}), ("no_norms", {"norms": False}), ("no_rope", {"rope": False}),
                     ("no_norms_no_rope", {"norms": False, "rope": False})):
        with torch.cuda.stream(st.torch_stream):
            step(st.sms, st.torch_stream, **kw)
            st.torch_stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st.torch_stream):
                step(st.sms, st.torch_stream, **kw)
        torch.cuda.synchronize()
        evs = []
        with torch.cuda.stream(st.torch_stream):
            for _ in range(8):
                lib.hold(st.torch_stream, 100_000)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                evs.append((a, b))
        torch.cuda.synchronize()
        out[name] = round(statistics.median(a.elapsed_time(b) * 1e3 for a, b in evs[1:]), 1)
    print(json.dumps(out), flush=True)
