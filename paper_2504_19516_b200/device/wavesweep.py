"""BASELINE config 3: wave quantization measured on the B200 vs the model.

For each prefill GEMM of a Llama-3-8B layer (qkv, o_proj, mlp_up_gate,
mlp_down at T tokens) and each partition size n on the green-context grid,
run the tcgen05 GEMM confined to n SMs with its persistent grid sized to n,
record every CTA's {smid, start, end} (%globaltimer), and compare

  measured idle  = 1 - sum_i busy_i / (n * span)
  predicted idle = wave_stats(tiles, 1, n).idle_ratio        (perf_model.py:157-169)

where `tiles` is the kernel's real work-unit count (128 x 256 output tiles)
and, for reference, the idle the reference's layer API predicts for its
nominal 128 x 128 grid (workload.py:169-209 grid rule).

    python -m paper_2504_19516_b200.device.wavesweep --out profiles/wave_sweep.json
"""

from __future__ import annotations

import argparse
import json

import torch

from ..perf_model import wave_stats
from ..workload import MODEL_PRESETS, layer_kernels
from . import lib
from .layer import LayerWeights
from .partition import DECODE, PREFILL, PartitionPool


def measure(pool: PartitionPool, x, w, y, epi, resid, n: int, reps: int = 3, tail: int = 0):
    """Measured idle of one GEMM launch on an n-SM partition, with the
    launch's plan (tiles, CTAs per tile) under the same tail mode.  tail = 0 (the
    default) times the plain persistent rounds that wave_stats describes;
    tail = 1 the stream-K tail (lib.set_gemm_tail), which spreads the last
    rounds' work over every pair."""
    st = pool.phase(DECODE, n) if n < pool.n else pool.full(PREFILL)
    times = torch.zeros(st.sms, 3, dtype=torch.int64, device=x.device)
    best = None
    lib.set_gemm_tail(tail)
    try:
        _, tiles, cpt = lib.gemm_plan(x.shape[0], w.shape[0], w.shape[1], st.sms)
        with torch.cuda.stream(st.torch_stream):
            for _ in range(reps):
                times.zero_()
                lib.hold(st.torch_stream, 100_000)
                lib.gemm_traced(x, w, y, times, epi, resid=resid, max_ctas=st.sms, stream=st.torch_stream)
                st.torch_stream.synchronize()
                t = times.cpu()
                t = t[t[:, 2] > 0]  # CTAs of this launch
                start, end = t[:, 1], t[:, 2]
                span = float(end.max() - start.min())
                busy = float((end - start).sum())
                idle = 1.0 - busy / (st.sms * span)
                if best is None or span < best[1]:
                    best = (idle, span, len(set(t[:, 0].tolist())))
    finally:
        lib.set_gemm_tail(-1)
    return best[0], best[1] * 1e-9, best[2], st.sms, tiles, cpt


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--tokens", default="1024,2048,4096")
    a = ap.parse_args(argv)
    m = MODEL_PRESETS["llama3-8b"]
    dev = torch.device("cuda", 0)
    pool = PartitionPool(0)
    gen = torch.Generator().manual_seed(0)
    W = LayerWeights.random(m, dev, gen)
    h, I = m.hidden, m.intermediate
    rows = []
    grid = list(range(16, pool.n, 8)) + [pool.n]
    for T in [int(s) for s in a.tokens.split(",")]:
        bf = dict(dtype=torch.bfloat16, device=dev)
        xh = torch.randn(T, h, **bf)
        xi = torch.randn(T, I, **bf)
        ref_grids = {k.name: k.grid_blocks for k in layer_kernels(m, "prefill", T, [T])}
        gemms = [("qkv", xh, W.w_qkv, torch.empty(T, m.qkv_out_dim, **bf), lib.EPI_STORE, None),
                 ("o_proj", xh, W.w_o, torch.empty(T, h, **bf), lib.EPI_RESID, xh),
                 ("mlp_up_gate", xh, W.w_ug, torch.empty(T, I, **bf), lib.EPI_SILU, None),
                 ("mlp_down", xi, W.w_down, torch.empty(T, h, **bf), lib.EPI_RESID, xh)]
        for name, x, w, y, epi, r in gemms:
            for n in grid:
                idle, span, sms_seen, n_real, tiles, cpt = measure(pool, x, w, y, epi, r, n)
                pred = wave_stats(tiles, 1, n_real // cpt)
                row = {"kernel": name, "T": T, "tiles": tiles, "n": n_real,
                       "predicted_idle": pred.idle_ratio, "waves": pred.waves, "tail_sms": pred.tail_sms,
                       "measured_idle": idle, "span_us": span * 1e6, "distinct_sms": sms_seen,
                       "reference_grid": ref_grids[name],
                       "reference_predicted_idle": wave_stats(ref_grids[name], 1, n_real).idle_ratio}
                rows.append(row)
                print(f"{name:12s} T={T:5d} tiles={tiles:4d} n={n_real:3d} waves={pred.waves:3d} "
                      f"pred={100 * pred.idle_ratio:5.1f}% meas={100 * idle:5.1f}% span={span * 1e6:8.1f}us",
                      flush=True)
    errs = [abs(r["measured_idle"] - r["predicted_idle"]) for r in rows]
    summary = {"points": len(rows), "mean_abs_err_pct": 100 * sum(errs) / len(errs),
               "max_abs_err_pct": 100 * max(errs)}
    print(json.dumps(summary))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"summary": summary, "rows": rows}, fh, indent=1)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
