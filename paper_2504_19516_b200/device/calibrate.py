"""Re-measure the estimator's tables on a B200 (SURVEY.md section 8 row a16,
"next" #3): the hardware half of `build_calibration_store`
(reference engine.py:238-260) and of the SRM's GpuSpec (perf_model.py:38-68).

    python -m paper_2504_19516_b200.device.calibrate --out calib/

Writes
  gpu.json           B200 GpuSpec: N, measured bf16 and HBM peaks, fitted n_d,
                     measured green-context repartition latency (reconfig_s)
  bandwidth.json     HBM GB/s vs SM count (green-context partitions) -- the
                     Fig. 6a curve behind D_p = D min(1, p / n_d)
  calibration.jsonl  alpha samples (prefill / decode, measured / SRM) and the
                     contention table, in the reference's JSONL format
                     (CalibrationStore.load_jsonl reads it)
  mape.json          estimator error on held-out points (Table 3 analogue):
                     36 prefill + 120 decode grid states + the decode SM axis

Also reachable as the reference's own command: `smshare calibrate --device
b200` (cli.py cmd_calibrate).
"""

from __future__ import annotations

import argparse
import json
from pathlib import Path

import torch

from ..engine import CalibrationBudget
from ..perf_model import CalibrationStore, PerfEstimator, b200_spec
from ..workload import MODEL_PRESETS
from . import lib
from .executor import B200Executor
from .partition import DECODE, PREFILL, PartitionPool

ROOT = Path(__file__).resolve().parents[2]


def bandwidth_curve(pool: PartitionPool, grid, nbytes: int = 1 << 30, reps: int = 3):
    buf = torch.ones(nbytes // 4, dtype=torch.float32, device="cuda")
    out = torch.zeros(4, device="cuda")
    rows = []
    for sms in grid:
        st = pool.phase(DECODE, sms)
        best = 0.0
        with torch.cuda.stream(st.torch_stream):
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                lib.hold(st.torch_stream, 100_000)
                a.record()
                lib.membw(buf, st.sms, 1, out, stream=st.torch_stream)
                b.record()
                torch.cuda.synchronize()
                best = max(best, nbytes / (a.elapsed_time(b) * 1e-3))
        rows.append((st.sms, best))
    return rows


def reconfig_latency(pool: PartitionPool, dm_a: int = 32, dm_b: int = 48, reps: int = 20) -> dict:
    """The reference's `reconfig_s` (engine.py:132; Table 6: 4.1
    us) on B200 green contexts: the gap between the end of a kernel on one
    decode partition and the start of the next kernel, measured with
    %globaltimer stamps, for (a) the next launch on the same stream, (b) on
    another stream of the same green context after an event, (c) on a
    different green-context partition after an event -- a repartition.
    reconfig_s = median(c) - median(a)."""
    import statistics

    a_st = pool.phase(DECODE, dm_a)
    b_st = pool.phase(DECODE, dm_b)
    same_ctx_other = pool.phase(PREFILL, pool.n - dm_a)  # the pair's other stream (same split)
    t1 = torch.zeros(a_st.sms, 3, dtype=torch.int64, device="cuda")
    t2 = torch.zeros(max(a_st.sms, b_st.sms), 3, dtype=torch.int64, device="cuda")

    def gap(first, second, cross: bool) -> float:
        ev = torch.cuda.Event()
        with torch.cuda.stream(first.torch_stream):
            lib.hold(first.torch_stream, 400_000)  # both launches queued before the first runs
            lib.probe(t1, first.sms, spin_ns=5000, stream=first.torch_stream)
            ev.record(first.torch_stream)
        st = second.torch_stream if cross else first.torch_stream
        with torch.cuda.stream(st):
            if cross:
                st.wait_event(ev)
            lib.probe(t2[:second.sms], second.sms, spin_ns=5000, stream=st)
        torch.cuda.synchronize()
        end_a = int(t1[:, 2].max())
        start_b = int(t2[:second.sms, 1].min())
        return (start_b - end_a) * 1e-9

    res = {}
    for name, (f, sec, cross) in {"same_stream": (a_st, a_st, False),
                                  "other_stream_same_split": (a_st, same_ctx_other, True),
                                  "other_partition": (a_st, b_st, True)}.items():
        gaps = [gap(f, sec, cross) for _ in range(reps)]
        res[name + "_us"] = 1e6 * statistics.median(gaps)
    res["reconfig_s"] = max(0.0, (res["other_partition_us"] - res["same_stream_us"]) * 1e-6)
    return res


def fit_n_d(curve, d_peak: float) -> int:
    """Least-squares n_d for D_p = d_peak * min(1, p / n_d)."""
    best, best_err = None, float("inf")
    for nd in range(1, max(s for s, _ in curve) + 1):
        err = sum((bw - d_peak * min(1.0, s / nd)) ** 2 for s, bw in curve)
        if err < best_err:
            best, best_err = nd, err
    return best


B200_BUDGET = dict(prefill_tokens=(512, 1024, 4096, 16384),
                  decode_tokens=(1024, 4096, 16384, 65536, 262144, 1048576, 2097152),
                  contention_prefill_lens=(1024, 4096, 16384))
# held-out points (disjoint from the budget's SM counts and token counts):
# 36 prefill and 120 decode states, plus the decode SM axis at the budget's
# token counts on every 8-SM share not in the budget
HELD_OUT = dict(prefill_seq_lens=(768, 2048, 3072, 6144, 8192, 12288), prefill_sms=(140, 124, 100, 68, 36, 20),
                decode_ctx_lens=(1536, 3072, 6144, 12288), decode_batch_sizes=(1, 8, 24, 64, 128, 192),
                decode_sms=(24, 40, 56, 96, 136))


def calibrate_b200(model, out: Path, quick: bool = False, pool: PartitionPool | None = None) -> dict:
    """The reference's calibration flow (cli.py:415-458 cmd_calibrate:
    build_calibration_store over a budget, then the decode SM-axis / decode
    grid / prefill grid MAPE helpers of engine.py:884-928) with the B200 as
    the oracle: every sample and every held-out point is a CUDA-event
    measurement of the real kernels on a green-context partition.  Also
    measures the GpuSpec half (HBM curve -> n_d, repartition latency).
    Writes gpu.json, bandwidth.json, calibration.jsonl, mape.json to `out`."""
    from ..engine import (build_calibration_store, canonical_decode_es, decode_mape_grid, decode_mape_sm_axis,
                          prefill_mape_grid)

    out.mkdir(parents=True, exist_ok=True)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    pool = pool or PartitionPool(0)
    N = pool.n
    grid = [8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 144, N]
    curve = bandwidth_curve(pool, grid)
    d_peak = max(bw for _, bw in curve)
    n_d = fit_n_d(curve, d_peak)
    gpu = b200_spec(c_peak=peaks.get("bf16_tflops", 1607.5) * 1e12, d_peak=d_peak, n_d=n_d, num_sms=N)
    rc = reconfig_latency(pool)
    (out / "gpu.json").write_text(json.dumps({**{k: getattr(gpu, k) for k in
                                                ("name", "num_sms", "c_peak", "d_peak", "w_peak", "n_d", "n_w")},
                                             "n_w_note": "preset: collective bandwidth vs SM count needs NVLink "
                                                         "peers (one GPU per gpurun call)",
                                             "reconfig_s": rc["reconfig_s"], "reconfig_gaps_us": rc},
                                             indent=2) + "\n")
    (out / "bandwidth.json").write_text(json.dumps({"sms_vs_bytes_per_s": curve, "n_d_fit": n_d}, indent=2) + "\n")

    ex = B200Executor(model, gpu, pool=pool, max_prefill_tokens=32768)
    b = dict(B200_BUDGET)
    if quick:
        b = dict(prefill_tokens=(1024, 4096), decode_tokens=(16384, 65536), contention_prefill_lens=(4096,))
    # SM axes: interior to every held-out point (prefill shares are N - 8k on
    # the green-context grid); the held-out shares are not sampled
    budget = CalibrationBudget(
        prefill_sms=(N, N - 16, N - 32, N - 64, N - 96, N - 120, N - 136) if not quick else (N, N - 64),
        prefill_tokens=b["prefill_tokens"],
        decode_sms=(8, 16, 32, 48, 64, 80, 112, N) if not quick else (16, 64), decode_tokens=b["decode_tokens"],
        contention_sms=(8, 16, 32, 64) if not quick else (16, 32),
        contention_prefill_lens=b["contention_prefill_lens"])
    store = build_calibration_store(ex, budget)
    store.dump_jsonl(out / "calibration.jsonl")

    est = PerfEstimator(model, gpu, CalibrationStore.load_jsonl(out / "calibration.jsonl"))
    h = HELD_OUT if not quick else dict(prefill_seq_lens=(2048,), prefill_sms=(116,), decode_ctx_lens=(3072,),
                                        decode_batch_sizes=(8,), decode_sms=(40,))
    sm_axis = [s for s in range(8, N, 8) if s not in budget.decode_sms]
    rep = {"device": "b200", "n_alpha_samples": len(store.alpha_samples),
           "n_contention_samples": len(store.contention_bw),
           "budget": {k: list(getattr(budget, k)) for k in ("prefill_sms", "prefill_tokens", "decode_sms",
                                                           "decode_tokens", "contention_sms",
                                                           "contention_prefill_lens")},
           "held_out": {k: list(v) for k, v in h.items()},
           "decode": {"sm_axis_mape": {str(tok): decode_mape_sm_axis(ex, est, tok, sm_axis if not quick else [40])
                                       for tok in budget.decode_tokens},
                      "grid_mape": decode_mape_grid(ex, est, h["decode_ctx_lens"], h["decode_batch_sizes"],
                                                    h["decode_sms"]),
                      "grid_points": len(h["decode_ctx_lens"]) * len(h["decode_batch_sizes"]) * len(h["decode_sms"])},
           "prefill": {"grid_mape": prefill_mape_grid(ex, est, h["prefill_seq_lens"], h["prefill_sms"]),
                       "grid_points": len(h["prefill_seq_lens"]) * len(h["prefill_sms"])},
           "n_d": n_d, "d_peak": d_peak}
    # per-point detail of the decode grid (measured, predicted), same states
    # as decode_mape_grid
    from ..perf_model import ExecutionState

    pts = []
    for cl in h["decode_ctx_lens"]:
        for bs in h["decode_batch_sizes"]:
            for dm in h["decode_sms"]:
                es = ExecutionState(decode_ctx_lens=tuple([cl] * bs), decode_sms=dm)
                pts.append([cl, bs, dm, ex.decode_step_s(es), est.decode_step_s([cl] * bs, dm)])
    rep["decode"]["grid_points_detail"] = pts
    axis = []
    for tok in budget.decode_tokens:
        for dm in (sm_axis if not quick else [40]):
            es = canonical_decode_es(tok, dm)
            axis.append([tok, dm, ex.decode_step_s(es), est.decode_step_s(list(es.decode_ctx_lens), dm)])
    rep["decode"]["sm_axis_points_detail"] = axis
    (out / "mape.json").write_text(json.dumps(rep, indent=2, sort_keys=True) + "\n")
    return rep


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="calib")
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args(argv)
    rep = calibrate_b200(MODEL_PRESETS[a.model], Path(a.out), a.quick)
    print(json.dumps({"n_d": rep["n_d"], "d_peak": rep["d_peak"], "prefill_grid_mape": rep["prefill"]["grid_mape"],
                      "decode_grid_mape": rep["decode"]["grid_mape"],
                      "decode_sm_axis_mape": rep["decode"]["sm_axis_mape"]}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
