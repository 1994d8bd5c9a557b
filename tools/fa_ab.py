"""Prefill attention TFLOP/s (causal, one sequence, Llama-3-8B heads) at
several T and grid sizes; run twice with HP_FA_PAIR=0/1 for A/B.

    HP_FA_PAIR=1 python tools/fa_ab.py
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

if os.environ.get("HP_LIB"):
    lib.load(os.environ["HP_LIB"])

dev = torch.device("cuda", 0)
Hq, Hkv, d = 32, 8, 128
out = {}
for T, sms in ((1024, 124), (2048, 132), (4096, 140), (4096, 148), (16384, 140), (16384, 148)):
    qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=dev).to(torch.bfloat16)
    q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    o = torch.empty(T, Hq * d, device=dev, dtype=torch.bfloat16)
    cu = torch.tensor([0, T], device=dev, dtype=torch.int32)

    def go():
        lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms)

    go()
    torch.cuda.synchronize()
    reps = max(3, int(2e10 / (2 * T * T * Hq * d)))
    ts = []
    for _ in range(3):
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            go()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3 / reps)
    t = sorted(ts)[1]
    out[f"T{T}_sms{sms}"] = round(2.0 * T * T * Hq * d / t / 1e12, 1)
# accuracy at one size (fp32 reference, chunked over query rows)
T = 2048
qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=dev).to(torch.bfloat16)
q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
o = torch.empty(T, Hq * d, device=dev, dtype=torch.bfloat16)
lib.prefill_attn(q, k, v, o, torch.tensor([0, T], device=dev, dtype=torch.int32), 1, T, Hq, Hkv, d,
                 1 / math.sqrt(d), max_ctas=148)
err = 0.0
for h in range(Hq):
    kh, vh = k.view(T, Hkv, d)[:, h // 4].float(), v.view(T, Hkv, d)[:, h // 4].float()
    sc = (q.view(T, Hq, d)[:, h].float() @ kh.T) / math.sqrt(d)
    sc = sc.masked_fill(torch.ones(T, T, device=dev, dtype=torch.bool).triu(1), float("-inf"))
    err = max(err, (o.view(T, Hq, d)[:, h].float() - sc.softmax(-1) @ vh).abs().max().item())
print(json.dumps({"lib": os.environ.get("HP_LIB", "default"), "HP_FA_PAIR": os.environ.get("HP_FA_PAIR", "auto"),
                  "tflops": out, "max_abs_err_T2048": err}))
