"""Decode attention GB/s (algorithmic K+V bytes) for several head shapes on
the full GPU; caches sized above L2 so back-to-back launches stream HBM.

    python tools/dattn_shapes.py
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_19516_b200.device import lib  # noqa: E402

SHAPES = [  # (name, Hq, Hkv, d)
    ("llama3-8b", 32, 8, 128), ("moe-a22b", 64, 4, 64), ("g8-d64", 32, 4, 64), ("llama3-70b/tp8", 8, 1, 128)]


def run(Hq, Hkv, d, B, ctx, sms=148, reps=10):
    dev = torch.device("cuda", 0)
    pages = -(-ctx // 64)
    nblk = B * pages
    kc = torch.randn(nblk, Hkv, 64, d, dtype=torch.bfloat16, device=dev)
    vc = torch.randn_like(kc)
    if os.environ.get("DA_SEQ"):  # measurement: pages laid out in order
        bt = torch.arange(nblk, device=dev).to(torch.int32).view(B, pages)
    else:
        bt = torch.randperm(nblk, device=dev).to(torch.int32).view(B, pages)
    cl = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    q = torch.randn(B, Hq * d, dtype=torch.bfloat16, device=dev)
    o = torch.empty_like(q)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 64) // 4 + 1, dtype=torch.float32, device=dev)

    stream = None
    if os.environ.get("DA_GREEN"):  # measurement: inside a green context of `sms` SMs
        from paper_2504_19516_b200.device.partition import DECODE, PartitionPool
        global _POOL
        if "_POOL" not in globals():
            _POOL = PartitionPool(0)
        st = _POOL.phase(DECODE, sms)
        stream = st.torch_stream

    def go():
        lib.decode_attn(q, kc, vc, bt, cl, o, Hq, Hkv, d, 64, 1 / math.sqrt(d), ws=ws, max_ctas=sms,
                        stream=stream)

    if stream is not None:
        with torch.cuda.stream(stream):
            return _timed(go, reps, B, ctx, Hkv, d, Hq)
    return _timed(go, reps, B, ctx, Hkv, d, Hq)


def _timed(go, reps, B, ctx, Hkv, d, Hq):
    go()
    ts = []
    for _ in range(3):
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            go()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps * 1e-3)
    t = sorted(ts)[1]
    nbytes = B * (ctx * 2 * Hkv * d * 2 + 2 * Hkv * d * 2 + 2 * Hq * d * 2)
    return nbytes / t / 1e9, t * 1e6, nbytes


if __name__ == "__main__":
    out = []
    for name, Hq, Hkv, d in SHAPES:
        for B, ctx in ((32, 2048), (128, 4096)):
            gbs, us, nb = run(Hq, Hkv, d, B, ctx)
            r = {"shape": name, "Hq": Hq, "Hkv": Hkv, "d": d, "B": B, "ctx": ctx, "MB": nb / 1e6, "us": us,
                 "GB/s": gbs, "launches": lib.decode_attn_launches(B, Hq, Hkv, d, -(-ctx // 64), 64, 148)}
            out.append(r)
            print(json.dumps(r), flush=True)
