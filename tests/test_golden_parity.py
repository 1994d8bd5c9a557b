"""Bit-exact parity of the host API against golden fixtures produced by the
REFERENCE implementation (tests/golden/make_golden.py imports
/root/reference/pkg/src/smshare).  Runs anywhere (the fixtures travel; the
reference does not).

Pins the integer outputs the north star requires to match exactly --
wave/tail/idle, SM-partition decisions (pm, dm, branch), schedule order and
batch membership -- plus the float estimator values (compared with ==, i.e.
identical IEEE doubles) that those decisions are derived from, at the B200
configuration (N = 148 SMs, sm_step 2 and 8).
"""

import hashlib
import json
import tempfile
from pathlib import Path

import pytest

from paper_2504_19516_b200 import engine as E
from paper_2504_19516_b200 import perf_model as P
from paper_2504_19516_b200 import scheduler as S
from paper_2504_19516_b200 import workload as W

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def gpu_of(d):
    return P.GpuSpec(**d)


MODELS = {"llama3-8b": W.MODEL_PRESETS["llama3-8b"], "llama3-70b": W.MODEL_PRESETS["llama3-70b"],
          "tiny": W.TINY_MODEL}


def store_of(d):
    st = P.CalibrationStore()
    for ph, sms, tok, v in d["alpha"]:
        st.alpha_samples[(ph, sms, tok)] = v
    for sms, sl, v in d["contention"]:
        st.contention_bw[(sms, sl)] = v
    return st


# --------------------------------------------------------------------- wave
def test_wave_stats_bit_exact():
    g = load("wave")
    for gg, b, n, waves, tail, idle in g["wave_stats"]:
        w = P.wave_stats(gg, b, n)
        assert (w.waves, w.tail_sms, w.idle_ratio) == (waves, tail, idle), (gg, b, n)


def test_wave_stats_native_library_bit_exact():
    """The C ABI's hp_wave_stats (host function, no GPU needed) agrees too."""
    from paper_2504_19516_b200.device import lib

    g = load("wave")
    for gg, b, n, waves, tail, idle in g["wave_stats"][::7]:
        assert lib.wave_stats(gg, b, n) == (waves, tail, idle)


def test_layer_grid_waves_on_partitions():
    g = load("wave")
    m = W.MODEL_PRESETS["llama3-8b"]
    for sl, name, grid, n, waves, tail, idle in g["layer_grids"]:
        k = {k.name: k for k in W.layer_kernels(m, "prefill", sl, [sl])}[name]
        assert k.grid_blocks == grid
        w = P.wave_stats(grid, 1, n)
        assert (w.waves, w.tail_sms, w.idle_ratio) == (waves, tail, idle)


# ------------------------------------------------------------------- layers
def test_layer_kernels_exact():
    g = load("layers")
    for case in g["layer_kernels"]:
        ks = W.layer_kernels(MODELS[case["model"]], case["phase"], case["new_tokens"],
                             case["ctx_lens"], case["prior_lens"])
        got = [[k.name, k.flops, k.mem_bytes, k.grid_blocks, k.blocks_per_sm] for k in ks]
        assert got == case["kernels"]
        assert W.batch_intensity(ks) == case["intensity"]


def test_hybrid_kernels_and_plans_exact():
    g = load("layers")
    for case in g["hybrid_kernels"]:
        ks = W.hybrid_kernels(MODELS[case["model"]], [tuple(c) for c in case["chunks"]], case["decode"])
        assert [[k.name, k.flops, k.mem_bytes, k.grid_blocks, k.blocks_per_sm] for k in ks] == case["kernels"]
    for sl, cs, ds, sizes, reloads, reproc in g["chunk_plans"]:
        plan = W.chunk_plan(sl, cs, ds)
        assert (list(plan.chunk_sizes), plan.reload_events, plan.reprocessed_tokens) == (sizes, reloads, reproc)
    for m, t, v in g["kv_bytes"]:
        assert W.kv_bytes(MODELS[m], t) == v


# ---------------------------------------------------------------- estimator
def test_estimator_exact():
    g = load("estimator")
    gpu = gpu_of(g["gpu"])
    store = store_of(g["store"])
    for row in g["rows"]:
        m = MODELS[row["model"]]
        pl, pm, dl, dm = row["es"]
        es = P.ExecutionState(tuple(pl), pm, tuple(dl), dm)
        e = P.estimate_latency(es, m, gpu, store)
        assert e.prefill_layer_s == row["prefill_layer_s"]
        assert e.decode_step_s == row["decode_step_s"]
        assert e.contention_fallback == row["fallback"]
        est = P.PerfEstimator(m, gpu, store)
        if "decode_step_s_co" in row:
            assert est.decode_step_s(list(dl), max(dm, 1), sum(pl)) == row["decode_step_s_co"]
        if "prefill_exec_s" in row:
            assert est.prefill_exec_s(list(pl), max(pm, 1)) == row["prefill_exec_s"]


def test_calibration_store_build_matches_reference():
    g = load("estimator")
    gpu = gpu_of(g["gpu"])
    budget = E.CalibrationBudget(prefill_sms=(40, 76, 108, 148), decode_sms=(8, 32, 64, 148),
                                 contention_sms=(8, 16, 32, 64, 104, 144))
    oracle = E.GroundTruthOracle(MODELS["llama3-8b"], gpu, E.OracleConfig())
    st = E.build_calibration_store(oracle, budget)
    ref = store_of(g["store"])
    assert st.alpha_samples == ref.alpha_samples
    assert st.contention_bw == ref.contention_bw


# ---------------------------------------------------------------- scheduler
def state_of(d):
    pl, pm, dl, dm = d["es"]
    reqs = {rid: S.ReqView(rid, arr, inp, ctx) for rid, arr, inp, ctx in d["requests"]}
    q, inflight, done = d["ps"]
    return S.SystemState(es=P.ExecutionState(tuple(pl), pm, tuple(dl), dm),
                         ps=S.PrefillState(list(q), list(inflight), done), requests=reqs,
                         sim_time=d["sim_time"], tpot_window=tuple(d["tpot_window"]),
                         decode_running=tuple(d["decode_running"]),
                         decode_ready=tuple(d["decode_ready"]),
                         kv_blocked=frozenset(d["kv_blocked"]),
                         decode_last_step_s=d["decode_last_step_s"])


def decision_dict(dc):
    return {"next_tasks": list(dc.next_tasks), "layers_to_run": dc.layers_to_run,
            "pm": dc.new_prefill_sms, "dm": dc.new_decode_sms, "suspended": dc.decode_suspended,
            "branch": dc.branch, "queue_order": list(dc.queue_order),
            "predicted_step_s": dc.predicted_step_s}


def test_scheduler_decisions_exact():
    g = load("decisions")
    gpu = gpu_of(g["gpu"])
    est = P.PerfEstimator(MODELS["llama3-8b"], gpu, store_of(g["store"]))
    branches = set()
    for rec in g["rows"]:
        cfg = S.SchedulerConfig(sm_step=rec["sm_step"])
        slo = S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=rec["tpot_s"])
        st = state_of(rec["state"])
        assert S.reorder_queue(st, slo, est) == rec["reorder"]
        dec = decision_dict(S.schedule_prefill(st, slo, est, cfg))
        assert dec == rec["prefill"]
        branches.add(dec["branch"])
        assert [[k, v] for k, v in st.ttft_estimates.items()] == rec["ttft_estimates"]
        assert list(S.set_balanced_sm(st, slo, est, cfg)) == rec["balanced"]
        assert S.min_decode_sms(st, slo, est, cfg) == rec["min_decode_sms"]
        assert decision_dict(S.schedule_decode(st, slo, est, cfg)) == rec["decode"]
        assert S.projected_suspension_p90(st, slo, est, cfg, [512, 1024]) == rec["suspension_p90"]
        if "handoff" in rec:
            assert decision_dict(S.transition_handoff(st, cfg, 148, 32)) == rec["handoff"]
    # the fixture exercises the interesting branches of Algorithm 1
    assert {"balanced", "reduce_prefill", "reduce_decode"} <= branches


# ------------------------------------------------------------------- engine
@pytest.mark.parametrize("idx", range(10))
def test_engine_runs_byte_identical(idx):
    g = load("runs")
    runs = g["runs"]
    if idx >= len(runs):
        pytest.skip("fewer runs in fixture")
    case = runs[idx]
    gpu = gpu_of(g["gpu"])
    budget = E.CalibrationBudget(**{k: tuple(v) if isinstance(v, list) else v for k, v in g["budget"].items()})
    slo = S.SloSpec(*g["slo"])
    pol = E.PolicySpec(case["policy"], chunk_size=1024, static_pm=108)
    cfg = E.SimConfig(gpu=gpu, model=MODELS[case["model"]], slo=slo,
                      sched=S.SchedulerConfig(sm_step=case["sm_step"]), policy=pol, seed=1,
                      noise_sigma=0.03, calibration=budget)
    trace = [W.Request(*r) for r in case["trace"]]
    rep = E.run(cfg, trace)
    assert rep.aggregates == case["aggregates"]
    log = [{k: e[k] for k in ("t", "pm", "dm", "branch", "batch", "layers") if k in e}
           for e in rep.decision_log]
    assert len(log) == case["n_decisions"]
    assert log[:400] == case["decisions"]
    assert [list(x) for x in rep.partition_timeline[:400]] == case["partition_timeline"]
    with tempfile.TemporaryDirectory() as tmp:
        paths = E.write_report(rep, tmp)
        dig = {k: hashlib.sha256(Path(p).read_bytes()).hexdigest() for k, p in sorted(paths.items())
               if k in case["digests"]}
    assert dig == case["digests"]
