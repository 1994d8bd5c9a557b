"""Real-time co-executed serving on the B200: the
reference's event loop on a wall clock, a whole model generating real
tokens, the decode step as one CUDA graph.

* tiny model (config 1 shapes), bullet policy: every request's freely
  generated tokens agree with the CPU oracle teacher-forced on them (only
  genuine bf16 ties may differ), every decode step is ONE graph launch, and
  every scheduling decision the engine took is reproduced by re-running the
  scheduler on the logged SystemState + calibration-store snapshot
  (tests/test_decision_replay.py re-runs the REFERENCE's scheduler on a
  committed log of such a run);
* nopartition policy runs the same loop on two full-device streams.
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from parity_harness import oracle_check_generation, tiny_weights  # noqa: E402

from paper_2504_19516_b200 import engine as E  # noqa: E402
from paper_2504_19516_b200 import perf_model as PM  # noqa: E402
from paper_2504_19516_b200 import scheduler as S  # noqa: E402
from paper_2504_19516_b200.device.layer import PAGE, LayerWeights  # noqa: E402
from paper_2504_19516_b200.device.partition import PartitionPool  # noqa: E402
from paper_2504_19516_b200.device.realtime import (RealtimeChunked, RealtimeSim, ServingModel,  # noqa: E402
                                                   kv_pages_for, state_from_json, store_from_json)
from paper_2504_19516_b200.device.split import b200_gpu, b200_store  # noqa: E402
from paper_2504_19516_b200.workload import TINY_MODEL, Request  # noqa: E402

DEV = torch.device("cuda", 0)
VOCAB = 1024
INPUTS = (17, 64, 200, 255, 256, 511, 512, 1000, 130, 700)
OUTPUTS = (12, 9, 16, 5, 20, 8, 13, 1, 17, 11)


@pytest.fixture(scope="module")
def tiny():
    m, Wl, embed, final_norm, lm_head = tiny_weights(0, VOCAB)

    def t(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(DEV)

    dW = [LayerWeights.from_numpy(DEV, w.w_qkv, w.w_o, w.w_gate, w.w_up, w.w_down, w.attn_norm, w.mlp_norm)
          for w in Wl]
    cfg = _cfg("bullet")
    srv = ServingModel(m, VOCAB, DEV, kv_pages=kv_pages_for(cfg, 64), max_prefill_tokens=8192,
                       max_pages_per_seq=-(-(max(INPUTS) + max(OUTPUTS) + 1) // PAGE), weights=dW,
                       embed=t(embed), final_norm=t(final_norm), lm_head=t(lm_head))
    return (m, Wl, embed, final_norm, lm_head), srv, PartitionPool(0)


def _cfg(policy):
    return E.SimConfig(gpu=b200_gpu(), model=TINY_MODEL, slo=S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.2),
                       sched=S.SchedulerConfig(sm_step=8, l_step=1), policy=E.PolicySpec(policy),
                       kv_pool_bytes=TINY_MODEL.weight_bytes() + (64 << 20), reconfig_s=0.0,
                       metadata_overhead_s=0.0, predict_overhead_s=0.0)


def _trace():
    return [Request(i, 0.004 * i, L, o) for i, (L, o) in enumerate(zip(INPUTS, OUTPUTS))]


def _prompts():
    rng = np.random.default_rng(7)
    return {i: rng.integers(0, VOCAB, L).astype(np.int32) for i, L in enumerate(INPUTS)}


@pytest.mark.parametrize("policy", ["bullet", "nopartition"])
def test_realtime_tiny_generates_oracle_tokens(tiny, policy):
    (m, Wl, embed, final_norm, lm_head), srv, pool = tiny
    prompts = _prompts()
    sim = RealtimeSim(_cfg(policy), _trace(), srv, pool, store=b200_store(), trace_decisions=True,
                      prompts=prompts)
    rep = sim.run()
    assert rep.aggregates["finished"] == len(INPUTS), rep.aggregates
    tot = {"matches": 0, "mismatches": 0, "tie_flips": 0}
    for rid, (L, o) in enumerate(zip(INPUTS, OUTPUTS)):
        toks = sim.generated[rid]
        assert len(toks) == o, (rid, len(toks), o)
        r = oracle_check_generation(m, Wl, embed, final_norm, lm_head, prompts[rid], toks)
        for k in tot:
            tot[k] += r[k]
        assert r["mismatches"] == 0, (rid, r)
    assert tot["tie_flips"] <= 2, tot
    # one graph launch per decode step; every decode step produced tokens
    assert sim.device_calls["decode_graph_replays"] == sim.device_calls["decode_steps"] > 0
    assert sim.host_busy_s > 0 and sim.wall_s >= sim.makespan * 0.5
    # the control plane's decisions, re-run on the logged inputs
    replayed = replay_decisions(sim.decisions, _cfg(policy))
    assert replayed["prefill"] + replayed["decode"] == len(sim.decisions)
    out = os.environ.get("HP_DECISIONS_OUT")
    if out and policy == "bullet":
        with open(out, "w") as fh:
            json.dump({"config": {"model": "tiny", "slo": [1.5e-3, 0.2], "sm_step": 8, "l_step": 1,
                                  "num_sms": 148, "gpu": _gpu_json()},
                       "decisions": sim.decisions}, fh)


def _gpu_json():
    g = b200_gpu()
    return {"name": g.name, "num_sms": g.num_sms, "c_peak": g.c_peak, "d_peak": g.d_peak, "w_peak": g.w_peak,
            "n_d": g.n_d, "n_w": g.n_w}


def replay_decisions(decisions, cfg, sched=S, perf_model=PM) -> dict:
    """Re-run `sched`'s schedule_prefill / transition_handoff /
    schedule_decode on each logged (SystemState, store) and require the
    logged decision."""
    n = {"prefill": 0, "decode": 0}
    L = cfg.model.num_layers
    for d in decisions:
        st = state_from_json(d["state"], (sched, perf_model))
        est = perf_model.PerfEstimator(cfg.model, cfg.gpu, store_from_json(d["store"], perf_model))
        if d["kind"] == "decode":
            got = sched.schedule_decode(st, cfg.slo, est, cfg.sched)
            assert list(got.next_tasks) == d["decision"]["batch"]
            assert got.predicted_step_s == d["decision"]["predicted_step_s"]
        else:
            handoff = (st.ps.in_flight and not st.ps.queue and cfg.sched.transition_layers > 0
                       and st.ps.layers_done >= L - cfg.sched.transition_layers
                       and (st.decode_running or st.decode_ready))
            got = (sched.transition_handoff(st, cfg.sched, cfg.gpu.num_sms, L) if handoff
                   else sched.schedule_prefill(st, cfg.slo, est, cfg.sched))
            want = d["decision"]
            assert (got.new_prefill_sms, got.new_decode_sms, got.branch, list(got.next_tasks),
                    got.layers_to_run) == (want["pm"], want["dm"], want["branch"], want["batch"],
                                           want["layers"]), (d["state"], want)
        n[d["kind"]] += 1
    return n


@pytest.mark.parametrize("chunk", [256, 64])
def test_realtime_tiny_chunked_generates_oracle_tokens(tiny, chunk):
    """The lockstep chunked baseline on the same model: hybrid batches with
    cached-prefix chunks and decode rows, real tokens vs the oracle."""
    (m, Wl, embed, final_norm, lm_head), srv, pool = tiny
    prompts = _prompts()
    cfg = _cfg("chunked")
    cfg.policy = E.PolicySpec("chunked", chunk_size=chunk)
    sim = RealtimeChunked(cfg, _trace(), srv, pool, prompts=prompts)
    rep = sim.run()
    assert rep.aggregates["finished"] == len(INPUTS), rep.aggregates
    flips = 0
    for rid, (L, o) in enumerate(zip(INPUTS, OUTPUTS)):
        toks = sim.generated[rid]
        assert len(toks) == o, (rid, len(toks), o)
        r = oracle_check_generation(m, Wl, embed, final_norm, lm_head, prompts[rid], toks)
        assert r["mismatches"] == 0, (rid, r)
        flips += r["tie_flips"]
    assert flips <= 2
    assert sim.device_calls["hybrid_iterations"] > len(INPUTS)
    assert len(sim.pages.free) == srv.kv_pages - 1  # every page returned


def test_realtime_llama3_8b_whole_model_serving():
    """Config 4's engine at full size (32 random-init Llama-3-8B layers, real
    tokens): a short Poisson-like burst through bullet; every decode step is
    one CUDA graph of the whole model on its partition, and requests of
    different lengths finish with their full output."""
    from paper_2504_19516_b200.workload import MODEL_PRESETS

    m = MODEL_PRESETS["llama3-8b"]
    cfg = E.SimConfig(gpu=b200_gpu(), model=m, slo=S.SloSpec(norm_ttft_s_per_token=3e-3, tpot_s=0.15),
                      sched=S.SchedulerConfig(sm_step=8), policy=E.PolicySpec("bullet"),
                      kv_pool_bytes=m.weight_bytes() + (4 << 30), reconfig_s=0.0,
                      metadata_overhead_s=0.0, predict_overhead_s=0.0)
    trace = [Request(i, 0.01 * i, L, o) for i, (L, o) in enumerate(((3000, 24), (700, 40), (5000, 8), (1500, 30)))]
    srv = ServingModel(m, 128256, DEV, kv_pages=kv_pages_for(cfg, 16), max_prefill_tokens=16384,
                       max_pages_per_seq=-(-(5000 + 40 + 1) // PAGE), max_batch=64, seed=3)
    sim = RealtimeSim(cfg, trace, srv, PartitionPool(0), store=b200_store())
    rep = sim.run()
    assert rep.aggregates["finished"] == len(trace), rep.aggregates
    for r in trace:
        toks = sim.generated[r.id]
        assert len(toks) == r.output_len and all(0 <= t < 128256 for t in toks)
    assert sim.device_calls["decode_graph_replays"] == sim.device_calls["decode_steps"] > 0
    assert sim.device_calls["prefill_steps"] >= len(trace) * m.num_layers // cfg.sched.l_step // 2
    assert rep.extended["ttft_p50_s"] > 0 and rep.extended["tpot_p50_ms"] > 0
    del srv
    torch.cuda.empty_cache()
