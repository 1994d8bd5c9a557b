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
  mape.json          estimator error on held-out points (Table 3 analogue)
"""

from __future__ import annotations

import argparse
import json
from pathlib import Path

import torch

from ..engine import CalibrationBudget, canonical_decode_es, mape
from ..perf_model import CalibrationStore, ExecutionState, PerfEstimator, b200_spec, update_online
from ..perf_model import srm_decode_step_s, srm_prefill_layer_s
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
                torch.cuda._sleep(100_000)
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
            torch.cuda._sleep(400_000)  # both launches queued before the first runs
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


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="calib")
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args(argv)
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    model = MODEL_PRESETS[a.model]
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    pool = PartitionPool(0)
    N = pool.n
    grid = [8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 144, N]
    curve = bandwidth_curve(pool, grid)
    d_peak = max(bw for _, bw in curve)
    n_d = fit_n_d(curve, d_peak)
    gpu = b200_spec(c_peak=peaks.get("bf16_tflops", 1607.5) * 1e12, d_peak=d_peak, n_d=n_d, num_sms=N)
    rc = reconfig_latency(pool)
    (out / "gpu.json").write_text(json.dumps({**{k: getattr(gpu, k) for k in
                                                ("name", "num_sms", "c_peak", "d_peak", "w_peak", "n_d", "n_w")},
                                             "reconfig_s": rc["reconfig_s"], "reconfig_gaps_us": rc},
                                             indent=2) + "\n")
    (out / "bandwidth.json").write_text(json.dumps({"sms_vs_bytes_per_s": curve, "n_d_fit": n_d}, indent=2) + "\n")

    ex = B200Executor(model, gpu, pool=pool, max_prefill_tokens=16384)
    budget = CalibrationBudget(
        prefill_sms=(N, N - 32, N - 64, N - 96) if not a.quick else (N, N - 64),
        prefill_tokens=(512, 1024, 4096, 16384) if not a.quick else (1024, 4096),
        decode_sms=(8, 16, 32, 64, N) if not a.quick else (16, 64),
        decode_tokens=(4096, 16384, 65536, 262144) if not a.quick else (16384, 65536),
        contention_sms=(8, 16, 32, 64) if not a.quick else (16, 32),
        contention_prefill_lens=(1024, 4096, 16384) if not a.quick else (4096,))
    store = CalibrationStore()
    for sms in budget.prefill_sms:
        for tok in budget.prefill_tokens:
            es = ExecutionState(prefill_lens=(tok,), prefill_sms=sms)
            update_online(store, "prefill", es, ex.prefill_layer_s(es), srm_prefill_layer_s(es, model, gpu))
    for sms in budget.decode_sms:
        for tok in budget.decode_tokens:
            es = canonical_decode_es(tok, sms)
            update_online(store, "decode", es, ex.decode_step_s(es), srm_decode_step_s(es, model, gpu))
    for sms in budget.contention_sms:
        for sl in budget.contention_prefill_lens:
            store.contention_bw[(sms, sl)] = ex.contention_bw(sms, sl)
    store.dump_jsonl(out / "calibration.jsonl")

    # held-out error of the calibrated estimator (Table 3 analogue)
    est = PerfEstimator(model, gpu, CalibrationStore.load_jsonl(out / "calibration.jsonl"))
    pre, dec = [], []
    for sms in ((N - 16, N - 48, N - 80) if not a.quick else (N - 32,)):
        for tok in ((768, 2048, 8192) if not a.quick else (2048,)):
            es = ExecutionState(prefill_lens=(tok,), prefill_sms=sms)
            pre.append((ex.prefill_layer_s(es), est.prefill_layer_s([tok], sms)))
    for sms in ((24, 48, 96) if not a.quick else (32,)):
        for tok in ((8192, 32768, 131072) if not a.quick else (32768,)):
            es = canonical_decode_es(tok, sms)
            dec.append((ex.decode_step_s(es), est.decode_step_s(list(es.decode_ctx_lens), sms)))
    rep = {"prefill_mape": mape(pre), "decode_mape": mape(dec), "prefill_pairs": pre, "decode_pairs": dec,
           "n_alpha_samples": len(store.alpha_samples), "n_contention_samples": len(store.contention_bw)}
    (out / "mape.json").write_text(json.dumps(rep, indent=2) + "\n")
    print(json.dumps({"n_d": n_d, "d_peak": d_peak, "prefill_mape": rep["prefill_mape"],
                      "decode_mape": rep["decode_mape"]}))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
