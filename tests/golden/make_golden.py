"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container (where the read-only reference is mounted):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package `smshare` (pkg/src/smshare) -- never this
repo's code -- and records inputs + outputs of the hot-path functions at the
B200 configuration (N = 148 SMs, sm_step 2 and 8) that the reference's own
tests do not cover:

  wave.json        wave_stats over a (g, b, n) grid incl. the config-3 sweep
                   (perf_model.py:157-169) and the per-kernel grids of
                   layer_kernels on the 8-SM partition grid
  layers.json      layer_kernels / hybrid_kernels FLOPs, bytes, grids
                   (workload.py:122-257) for llama3-8b, llama3-70b, tiny
  estimator.json   estimate_latency / PerfEstimator on random states
                   (perf_model.py:386-481)
  decisions.json   schedule_prefill / set_balanced_sm / min_decode_sms /
                   schedule_decode / transition_handoff on seeded random
                   SystemStates (scheduler.py:111-409)
  runs.json        full engine.run() decision logs + report digests on
                   config-1 / config-4 style traces (engine.py:345-866)

JSON floats round-trip exactly (repr), so the fixtures pin bit-exact parity.
The fixtures travel to the GPU box; this script does not.
"""

from __future__ import annotations

import hashlib
import json
import random
import sys
import tempfile
from pathlib import Path

import smshare
from smshare import engine as E
from smshare import perf_model as P
from smshare import scheduler as S
from smshare import workload as W

assert "/root/reference" in smshare.__file__, f"must import the reference, got {smshare.__file__}"

OUT = Path(__file__).resolve().parent

B200 = P.GpuSpec("B200", num_sms=148, c_peak=1607.5e12, d_peak=6540.8e9, w_peak=900e9,
                 n_d=40, n_w=8)
TINY = W.ModelSpec("tiny", num_layers=2, hidden=256, num_heads=4, num_kv_heads=2,
                   head_dim=64, intermediate=768)
MODELS = {"llama3-8b": W.MODEL_PRESETS["llama3-8b"], "llama3-70b": W.MODEL_PRESETS["llama3-70b"],
          "tiny": TINY}
B200_BUDGET = E.CalibrationBudget(
    prefill_sms=(40, 76, 108, 148), decode_sms=(8, 32, 64, 148),
    contention_sms=(8, 16, 32, 64, 104, 144))


def model_dict(m):
    return {k: getattr(m, k) for k in ("name", "num_layers", "hidden", "num_heads", "num_kv_heads",
                                        "head_dim", "intermediate", "dtype_bytes",
                                        "activated_fraction")}


def gpu_dict(g):
    return {k: getattr(g, k) for k in ("name", "num_sms", "c_peak", "d_peak", "w_peak", "n_d", "n_w")}


def kd(k):
    return [k.name, k.flops, k.mem_bytes, k.grid_blocks, k.blocks_per_sm]


def gen_wave():
    rows = []
    for n in (78, 108, 132, 148):
        for b in (1, 2, 3, 4):
            for g in list(range(1, 400)) + [1000, 1792, 3456, 6144, 65536]:
                w = P.wave_stats(g, b, n)
                rows.append([g, b, n, w.waves, w.tail_sms, w.idle_ratio])
    parts = list(range(8, 148, 8)) + [148]
    kern = []
    for sl in (1024, 2048, 4096, 16384):
        for k in W.layer_kernels(MODELS["llama3-8b"], "prefill", sl, [sl]):
            for n in parts:
                w = P.wave_stats(k.grid_blocks, k.blocks_per_sm, n)
                kern.append([sl, k.name, k.grid_blocks, n, w.waves, w.tail_sms, w.idle_ratio])
    return {"wave_stats": rows, "layer_grids": kern}


def gen_layers():
    rng = random.Random(7)
    cases = []
    for mname, m in MODELS.items():
        for sl in (1, 17, 128, 1000, 1024, 2048, 4096, 16384):
            cases.append(["prefill", mname, sl, [sl], None])
        for _ in range(20):
            lens = [rng.randint(1, 5000) for _ in range(rng.randint(1, 6))]
            priors = [rng.randint(0, 8000) for _ in lens] if rng.random() < 0.5 else None
            cases.append(["prefill", mname, sum(lens), lens, priors])
        for bs in (1, 8, 32, 128):
            ctxs = [rng.randint(1, 9000) for _ in range(bs)]
            cases.append(["decode", mname, bs, ctxs, None])
        cases.append(["decode", mname, 32, [2048] * 32, None])
    out = []
    for phase, mname, nt, lens, priors in cases:
        ks = W.layer_kernels(MODELS[mname], phase, nt, lens, priors)
        out.append({"phase": phase, "model": mname, "new_tokens": nt, "ctx_lens": lens,
                    "prior_lens": priors, "kernels": [kd(k) for k in ks],
                    "intensity": W.batch_intensity(ks)})
    hyb = []
    for _ in range(30):
        mname = rng.choice(list(MODELS))
        chunks = [(rng.randint(1, 2048), rng.randint(0, 8000)) for _ in range(rng.randint(0, 3))]
        dec = [rng.randint(1, 8000) for _ in range(rng.randint(0 if chunks else 1, 40))]
        ks = W.hybrid_kernels(MODELS[mname], chunks, dec)
        hyb.append({"model": mname, "chunks": chunks, "decode": dec, "kernels": [kd(k) for k in ks]})
    plans = [[sl, cs, ds, P.__name__ and list(W.chunk_plan(sl, cs, ds).chunk_sizes),
              W.chunk_plan(sl, cs, ds).reload_events, W.chunk_plan(sl, cs, ds).reprocessed_tokens]
             for sl, cs, ds in ((16384, 1024, 32), (16384, 2048, 0), (5000, 512, 100), (7, 8, 7))]
    return {"layer_kernels": out, "hybrid_kernels": hyb, "chunk_plans": plans,
            "kv_bytes": [[m, t, W.kv_bytes(MODELS[m], t)] for m in MODELS for t in (0, 1, 4096)]}


def store_dict(store):
    return {"alpha": [[k[0], k[1], k[2], v] for k, v in sorted(store.alpha_samples.items())],
            "contention": [[k[0], k[1], v] for k, v in sorted(store.contention_bw.items())]}


def make_store():
    oracle = E.GroundTruthOracle(MODELS["llama3-8b"], B200, E.OracleConfig())
    return E.build_calibration_store(oracle, B200_BUDGET)


def gen_estimator():
    store = make_store()
    rng = random.Random(11)
    rows = []
    for mname in ("llama3-8b", "tiny"):
        m = MODELS[mname]
        est = P.PerfEstimator(m, B200, store)
        for _ in range(60):
            pl = tuple(rng.randint(1, 16384) for _ in range(rng.randint(0, 3)))
            dl = tuple(rng.randint(1, 8192) for _ in range(rng.choice([0, 1, 8, 32, 64])))
            pm = rng.choice([0, 8, 40, 100, 116, 140, 148]) if pl else 0
            dm = rng.choice([8, 16, 32, 48, 148]) if dl else 0
            if not ((pl and pm) or (dl and dm)):
                continue
            es = P.ExecutionState(pl, pm, dl, dm)
            e = P.estimate_latency(es, m, B200, store)
            row = {"model": mname, "es": [list(pl), pm, list(dl), dm],
                   "prefill_layer_s": e.prefill_layer_s, "decode_step_s": e.decode_step_s,
                   "fallback": e.contention_fallback}
            if dl:
                row["decode_step_s_co"] = est.decode_step_s(list(dl), max(dm, 1), sum(pl))
            if pl:
                row["prefill_exec_s"] = est.prefill_exec_s(list(pl), max(pm, 1))
            rows.append(row)
    return {"gpu": gpu_dict(B200), "store": store_dict(store), "rows": rows}


def state_dict(st):
    return {"es": [list(st.es.prefill_lens), st.es.prefill_sms, list(st.es.decode_ctx_lens),
                   st.es.decode_sms],
            "ps": [list(st.ps.queue), list(st.ps.in_flight), st.ps.layers_done],
            "requests": [[r.id, r.arrival_s, r.input_len, r.ctx_len] for r in st.requests.values()],
            "sim_time": st.sim_time, "tpot_window": list(st.tpot_window),
            "decode_running": list(st.decode_running), "decode_ready": list(st.decode_ready),
            "kv_blocked": sorted(st.kv_blocked), "decode_last_step_s": st.decode_last_step_s}


def random_state(rng, n):
    reqs = {}
    rid = 0

    def new(arrival_max, ctx=0):
        nonlocal rid
        r = S.ReqView(rid, rng.uniform(0, arrival_max), rng.randint(16, 8192), ctx)
        reqs[rid] = r
        rid += 1
        return r.id

    now = rng.uniform(0.5, 20.0)
    queue = [new(now) for _ in range(rng.randint(0, 8))]
    inflight = [new(now) for _ in range(rng.randint(0, 2))] if rng.random() < 0.6 else []
    running = [new(now, rng.randint(1, 9000)) for _ in range(rng.choice([0, 0, 4, 16, 32]))]
    ready = [new(now, 0) for _ in range(rng.choice([0, 0, 1, 3]))]
    dm = rng.choice([0, 8, 16, 24, 32, 48, 64, 96, 144]) if (running or rng.random() < 0.3) else 0
    dm = min(dm, n - 4)
    pm = n - dm if rng.random() < 0.9 else rng.choice([0, n])
    es = P.ExecutionState(tuple(reqs[r].input_len for r in inflight), pm,
                          tuple(reqs[r].ctx_len for r in running), dm)
    window = [rng.uniform(0.005, 0.4) for _ in range(rng.choice([0, 3, 20, 64]))]
    kv_blocked = frozenset(r for r in queue + ready if rng.random() < 0.15)
    return S.SystemState(es=es, ps=S.PrefillState(queue, inflight, rng.randint(0, 31) if inflight else 0),
                         requests=reqs, sim_time=now, tpot_window=tuple(window),
                         decode_running=tuple(running), decode_ready=tuple(ready),
                         kv_blocked=kv_blocked, decode_last_step_s=now - rng.uniform(0, 0.5))


def decision_dict(d):
    return {"next_tasks": list(d.next_tasks), "layers_to_run": d.layers_to_run,
            "pm": d.new_prefill_sms, "dm": d.new_decode_sms, "suspended": d.decode_suspended,
            "branch": d.branch, "queue_order": list(d.queue_order),
            "predicted_step_s": d.predicted_step_s}


def gen_decisions():
    store = make_store()
    est = P.PerfEstimator(MODELS["llama3-8b"], B200, store)
    rng = random.Random(2024)
    rows = []
    for sm_step in (2, 8):
        cfg = S.SchedulerConfig(sm_step=sm_step)
        for tpot_ms in (20.0, 60.0, 200.0):
            slo = S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=tpot_ms * 1e-3)
            for _ in range(60 if sm_step == 8 else 40):
                st = random_state(rng, B200.num_sms)
                rec = {"sm_step": sm_step, "tpot_s": slo.tpot_s, "state": state_dict(st)}
                rec["reorder"] = S.reorder_queue(st, slo, est)
                rec["prefill"] = decision_dict(S.schedule_prefill(st, slo, est, cfg))
                rec["ttft_estimates"] = [[k, v] for k, v in st.ttft_estimates.items()]
                rec["balanced"] = list(S.set_balanced_sm(st, slo, est, cfg))
                rec["min_decode_sms"] = S.min_decode_sms(st, slo, est, cfg)
                rec["decode"] = decision_dict(S.schedule_decode(st, slo, est, cfg))
                rec["suspension_p90"] = S.projected_suspension_p90(st, slo, est, cfg, [512, 1024])
                if st.ps.in_flight and st.ps.layers_done >= 32 - cfg.transition_layers:
                    rec["handoff"] = decision_dict(S.transition_handoff(st, cfg, 148, 32))
                rows.append(rec)
    return {"gpu": gpu_dict(B200), "store": store_dict(store), "rows": rows}


def digest_report(rep, tmp):
    paths = E.write_report(rep, tmp)
    return {k: hashlib.sha256(Path(p).read_bytes()).hexdigest() for k, p in sorted(paths.items())}


def gen_runs():
    out = []
    tiny_trace = [W.Request(0, 0.0, 1024, 16)] + [
        W.Request(i + 1, 0.001 * (i + 1), c, 16) for i, c in enumerate((17, 64, 128, 255, 256, 511, 512, 1000))]
    ins = W.LengthDist("uniform", lo=512, hi=8192)
    outs = W.TRACE_PRESETS["sharegpt-like"][1]
    serving = W.gen_poisson_trace(4.0, 20.0, ins, outs, seed=3)
    cases = [("tiny", tiny_trace), ("llama3-8b", serving)]
    slo = S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.05)
    for mname, trace in cases:
        for sm_step in (2, 8):
            for policy in ("bullet", "nopartition", "static", "chunked"):
                if sm_step == 8 and policy in ("nopartition", "chunked"):
                    continue
                pol = E.PolicySpec(policy, chunk_size=1024, static_pm=108)
                cfg = E.SimConfig(gpu=B200, model=MODELS[mname], slo=slo,
                                  sched=S.SchedulerConfig(sm_step=sm_step), policy=pol,
                                  seed=1, noise_sigma=0.03, calibration=B200_BUDGET)
                rep = E.run(cfg, trace)
                with tempfile.TemporaryDirectory() as tmp:
                    dig = digest_report(rep, tmp)
                log = [{k: e[k] for k in ("t", "pm", "dm", "branch", "batch", "layers") if k in e}
                       for e in rep.decision_log]
                out.append({"model": mname, "sm_step": sm_step, "policy": policy,
                            "trace": [[r.id, r.arrival_s, r.input_len, r.output_len] for r in trace],
                            "aggregates": rep.aggregates, "digests": dig,
                            "decisions": log[:400], "n_decisions": len(log),
                            "partition_timeline": [list(x) for x in rep.partition_timeline[:400]]})
    return {"gpu": gpu_dict(B200), "slo": [slo.norm_ttft_s_per_token, slo.tpot_s],
            "budget": {k: list(v) if isinstance(v, tuple) else v
                       for k, v in B200_BUDGET.__dict__.items()}, "runs": out}


def main():
    sizes = {}
    for name, fn in (("wave", gen_wave), ("layers", gen_layers), ("estimator", gen_estimator),
                     ("decisions", gen_decisions), ("runs", gen_runs)):
        data = fn()
        data["_generated_by"] = "tests/golden/make_golden.py from /root/reference/pkg/src/smshare"
        path = OUT / f"{name}.json"
        path.write_text(json.dumps(data, separators=(",", ":")) + "\n")
        sizes[name] = path.stat().st_size
    print(json.dumps(sizes))


if __name__ == "__main__":
    sys.exit(main())
