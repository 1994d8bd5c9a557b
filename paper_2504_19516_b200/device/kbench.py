"""Per-kernel microbenchmarks (CUDA events, L2 flushed between iterations).

    python -m paper_2504_19516_b200.device.kbench [--json out.json]

Prints achieved TFLOP/s (GEMM, prefill attention) or GB/s (decode attention,
decode GEMMs) against MEASURED_PEAKS.json for the Llama-3-8B layer shapes.
"""

from __future__ import annotations

import argparse
import json
import math
import sys

import torch

from . import lib

DEV = torch.device("cuda", 0)


def timeit(fn, iters=20, warmup=3, flush=True, stream=None):
    # L2 flush by READING a buffer larger than L2 (a write-based flush would
    # leave ~126 MB of dirty lines to be written back inside the timed kernel)
    flush_buf = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=DEV) if flush else None
    st = stream or torch.cuda.current_stream()
    times = []
    with torch.cuda.stream(st):
        for i in range(warmup + iters):
            if flush_buf is not None:
                flush_buf.sum()
            # keep the GPU busy while the host enqueues the timed launch, so
            # host-side launch latency never lands between the two events
            torch.cuda._sleep(100_000)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            if i >= warmup:
                times.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(x.elapsed_time(y) for x, y in times)
    return ms[len(ms) // 2] * 1e-3


def bench_gemm(T, N, K, epi, sms, results):
    x = torch.randn(T, K, device=DEV).to(torch.bfloat16)
    w = lib.tile_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
    outN = N // 2 if epi == lib.EPI_SILU else N
    y = torch.empty(T, outN, device=DEV, dtype=torch.bfloat16)
    r = torch.randn(T, outN, device=DEV).to(torch.bfloat16) if epi == lib.EPI_RESID else None
    t = timeit(lambda: lib.gemm(x, w, y, epi, resid=r, max_ctas=sms))
    tf = 2.0 * T * N * K / t / 1e12
    ref = None
    if sms == 148 and epi == lib.EPI_STORE:
        tr = timeit(lambda: torch.matmul(x, w.T, out=y))
        ref = 2.0 * T * N * K / tr / 1e12
    results.append({"kernel": "gemm", "T": T, "N": N, "K": K, "epi": epi, "sms": sms,
                    "us": t * 1e6, "tflops": tf, "cublas_tflops": ref})
    print(f"gemm T={T:6d} N={N:6d} K={K:6d} epi={epi} sms={sms:3d}: {t*1e6:9.1f} us "
          f"{tf:8.1f} TFLOP/s" + (f"  (torch/cuBLAS {ref:.1f})" if ref else ""), flush=True)


def bench_gemm_swap(T, N, K, epi, sms, results):
    x = torch.randn(T, K, device=DEV).to(torch.bfloat16)
    w = lib.tile_weight((torch.randn(N, K, device=DEV) * 0.02).to(torch.bfloat16))
    outN = N // 2 if epi == lib.EPI_SILU else N
    y = torch.empty(T, outN, device=DEV, dtype=torch.bfloat16)
    r = torch.randn(T, outN, device=DEV).to(torch.bfloat16) if epi == lib.EPI_RESID else None
    bn = 32 if T <= 32 else 64 if T <= 64 else 128 if T <= 128 else 256
    ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, sms) // 4, device=DEV)
    cnt = torch.zeros((N // 128) * (-(-T // bn)), device=DEV, dtype=torch.int32)
    t = timeit(lambda: lib.gemm_swap(x, w, y, ws, cnt, epi, resid=r, max_ctas=sms))
    gbs = (N * K * 2 + T * K * 2 + T * outN * 2) / t / 1e9
    results.append({"kernel": "gemm_swap", "T": T, "N": N, "K": K, "epi": epi, "sms": sms,
                    "us": t * 1e6, "gbs": gbs})
    print(f"gemm_swap T={T:4d} N={N:6d} K={K:6d} epi={epi} sms={sms:3d}: {t*1e6:8.1f} us "
          f"{gbs:8.1f} GB/s (weights streamed)", flush=True)


def bench_decode_attn(B, ctx, Hq, Hkv, sms, results):
    d, page = 128, 64
    pages = -(-ctx // page)
    nblk = B * pages
    kc = torch.randn(nblk, Hkv, page, d, device=DEV).to(torch.bfloat16)
    vc = torch.randn(nblk, Hkv, page, d, device=DEV).to(torch.bfloat16)
    bt = torch.randperm(nblk, device=DEV).to(torch.int32).view(B, pages)
    q = torch.randn(B, Hq * d, device=DEV).to(torch.bfloat16)
    out = torch.empty_like(q)
    cl = torch.full((B,), ctx, device=DEV, dtype=torch.int32)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 512) // 4, device=DEV)
    t = timeit(lambda: lib.decode_attn(q, kc, vc, bt, cl, out, Hq, Hkv, d, page, 1 / math.sqrt(d),
                                       ws=ws, max_ctas=sms))
    nbytes = B * (ctx * 2 * Hkv * d * 2 + 2 * Hkv * d * 2 + 2 * Hq * d * 2)
    gbs = nbytes / t / 1e9
    results.append({"kernel": "decode_attn", "B": B, "ctx": ctx, "sms": sms, "us": t * 1e6,
                    "gbs": gbs, "bytes": nbytes})
    print(f"decode_attn B={B} ctx={ctx} sms={sms:3d}: {t*1e6:8.1f} us {gbs:8.1f} GB/s", flush=True)


def bench_prefill_attn(T, Hq, Hkv, sms, results):
    d = 128
    qkv = torch.randn(T, (Hq + 2 * Hkv) * d, device=DEV).to(torch.bfloat16)
    q, k, v = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    cu = torch.tensor([0, T], device=DEV, dtype=torch.int32)
    t = timeit(lambda: lib.prefill_attn(q, k, v, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms))
    fl = 2.0 * T * T * Hq * d  # causal: 4 T^2 h / 2
    results.append({"kernel": "prefill_attn", "T": T, "sms": sms, "us": t * 1e6,
                    "tflops": fl / t / 1e12})
    print(f"prefill_attn T={T:6d} sms={sms:3d}: {t*1e6:9.1f} us {fl/t/1e12:8.1f} TFLOP/s", flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args(argv)
    res = []
    h, qkv, inter = 4096, 6144, 14336
    for T in ([1024, 4096] if a.quick else [1024, 2048, 4096, 16384]):
        bench_gemm(T, qkv, h, lib.EPI_STORE, 148, res)
        bench_gemm(T, h, h, lib.EPI_RESID, 148, res)
        bench_gemm(T, 2 * inter, h, lib.EPI_SILU, 148, res)
        bench_gemm(T, h, inter, lib.EPI_RESID, 148, res)
        bench_prefill_attn(T, 32, 8, 148, res)
    bench_gemm(4096, 2 * inter, h, lib.EPI_STORE, 148, res)
    for sms in (148, 116, 64):
        bench_gemm(4096, 2 * inter, h, lib.EPI_SILU, sms, res)
    for sms in ([148, 32] if a.quick else [148, 96, 64, 48, 32, 16]):
        bench_decode_attn(32, 2048, 32, 8, sms, res)
    for sms in (148, 64, 32):
        bench_gemm_swap(32, qkv, h, lib.EPI_STORE, sms, res)
        bench_gemm_swap(32, h, h, lib.EPI_RESID, sms, res)
        bench_gemm_swap(32, 2 * inter, h, lib.EPI_SILU, sms, res)
        bench_gemm_swap(32, h, inter, lib.EPI_RESID, sms, res)
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
