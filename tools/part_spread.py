"""Contiguous vs spread green-context decode shares (HP_PART_SPREAD=1):
decode-attention GB/s on the dm-SM side alone and beside the prefill
up-gate GEMM on the other side; SM ids of each side.

    HP_PART_SPREAD=0|1 python tools/part_spread.py [dm ...]
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402
from paper_2504_19516_b200.device.layer import LayerWeights  # noqa: E402
from paper_2504_19516_b200.workload import MODEL_PRESETS  # noqa: E402

dev = torch.device("cuda", 0)
m = MODEL_PRESETS["llama3-8b"]
B, ctx, Hq, Hkv, d = 32, 2048, 32, 8, 128
pages = ctx // 64
nblk = B * pages
kc = torch.randn(nblk, Hkv, 64, d, dtype=torch.bfloat16, device=dev)
vc = torch.randn_like(kc)
bt = torch.randperm(nblk, device=dev).to(torch.int32).view(B, pages)
cl = torch.full((B,), ctx, dtype=torch.int32, device=dev)
q = torch.randn(B, Hq * d, dtype=torch.bfloat16, device=dev)
o = torch.empty_like(q)
ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 64) // 4 + 1, dtype=torch.float32, device=dev)
nbytes = B * (ctx * 2 * Hkv * d * 2 + 2 * Hkv * d * 2 + 2 * Hq * d * 2)
g = torch.Generator(device=dev)
g.manual_seed(0)
W = LayerWeights.random_device(m, dev, g)
T = 4096
x = torch.randn(T, m.hidden, dtype=torch.bfloat16, device=dev)
y = torch.empty(T, m.intermediate, dtype=torch.bfloat16, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


for dm in [int(a) for a in sys.argv[1:]] or [16, 32, 48, 64]:
    part = lib.Partition(dm)
    ds, ps = part.stream(1), part.stream(0)
    sms = {}
    for ph, st in ((0, ps), (1, ds)):
        buf = torch.zeros(4 * 148, 3, dtype=torch.int64, device=dev)
        lib.probe(buf, 4 * 148, spin_ns=30000, stream=st)
        st.synchronize()
        sms[ph] = sorted(set(buf[:, 0].tolist()))

    def attn():
        lib.decode_attn(q, kc, vc, bt, cl, o, Hq, Hkv, d, 64, 1 / math.sqrt(d), ws=ws, max_ctas=part.decode_sms,
                        stream=ds)

    def gemm():
        lib.gemm(x, W.w_ug, y, lib.EPI_SILU, max_ctas=part.prefill_sms, stream=ps)

    res = {}
    for mode in ("alone", "corun"):
        with torch.cuda.stream(ds):
            attn()
        torch.cuda.synchronize()
        a0, a1, g0, g1 = ev(), ev(), ev(), ev()
        torch.cuda._sleep(200000)
        start = ev()
        start.record()
        ds.wait_event(start)
        ps.wait_event(start)
        if mode == "corun":
            with torch.cuda.stream(ps):
                g0.record(ps)
                for _ in range(6):
                    gemm()
                g1.record(ps)
        with torch.cuda.stream(ds):
            a0.record(ds)
            for _ in range(20):
                attn()
            a1.record(ds)
        torch.cuda.synchronize()
        res[mode] = nbytes * 20 / (a0.elapsed_time(a1) * 1e-3) / 1e9
        if mode == "corun":
            res["gemm_tflops"] = 6 * 4.0 * T * m.intermediate * m.hidden / (g0.elapsed_time(g1) * 1e-3) / 1e12
            res["attn_window_overlaps_gemm"] = a1.elapsed_time(g1) > 0
    print(json.dumps({"spread": os.environ.get("HP_PART_SPREAD", "0"), "dm": dm, "decode_sms": part.decode_sms,
                      "prefill_sms": part.prefill_sms, "attn_gbs_alone": round(res["alone"]),
                      "attn_gbs_corun": round(res["corun"]), "gemm_tflops_corun": round(res["gemm_tflops"]),
                      "decode_smids": sms[1][:64]}), flush=True)
