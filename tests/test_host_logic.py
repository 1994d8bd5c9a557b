"""Host-side logic of the round-2 paths, on CPU (no device calls):
the estimator's config-2 split, the co-run decode cadence, the real-time
engine's page pool / buckets / KV sizing, the decision-fixture codecs and
the incremental calibration-store axes."""

import random

import pytest

from paper_2504_19516_b200 import engine as E
from paper_2504_19516_b200 import perf_model as PM
from paper_2504_19516_b200 import scheduler as S
from paper_2504_19516_b200.device.corun import decode_schedule
from paper_2504_19516_b200.device.realtime import (BUCKETS, PageAllocator, bucket_of, delta_decode, delta_encode,
                                                   kv_pages_for, state_from_json, state_to_json, store_from_json)
from paper_2504_19516_b200.device.split import b200_gpu, b200_store, corun_state, estimator_split
from paper_2504_19516_b200.errors import InvalidArgumentError
from paper_2504_19516_b200.workload import MODEL_PRESETS, kv_bytes

M = MODEL_PRESETS["llama3-8b"]


def _ts_slo(T, t_p, t_d):
    ts = t_p + t_d
    return S.SloSpec(norm_ttft_s_per_token=M.num_layers * ts / T, tpot_s=M.num_layers * ts)


def test_estimator_split_follows_algorithm_1_on_the_b200_store():
    gpu, store = b200_gpu(), b200_store()
    # loose TPOT (long prefill layers): decode gets the minimum share
    r = estimator_split(M, 16384, [2048] * 32, _ts_slo(16384, 6.4e-3, 1.2e-4), gpu, store)
    assert (r["pm"], r["dm"]) == (140, 8) and r["pm"] + r["dm"] == gpu.num_sms
    # tight TPOT (short prefill layers): decode needs more SMs
    r2 = estimator_split(M, 1024, [2048] * 32, _ts_slo(1024, 3.4e-4, 1.1e-4), gpu, store)
    assert r2["dm"] > 8 and r2["dm"] % 8 == 0
    for x in (r, r2):
        assert x["branch"] in ("min_decode_sms", "set_balanced_sm")
        assert x["predicted_prefill_layer_s"] > 0 and x["predicted_decode_layer_s"] > 0
    # the decision is the reference functions' own: min_decode_sms on the same state
    st = corun_state(1024, [2048] * 32, gpu.num_sms, dm0=8)
    est = PM.PerfEstimator(M, gpu, store)
    dm = S.min_decode_sms(st, _ts_slo(1024, 3.4e-4, 1.1e-4), est, S.SchedulerConfig(sm_step=8))
    if r2["branch"] == "min_decode_sms":
        assert r2["dm"] == dm


@pytest.mark.parametrize("ratio", [1.0, 1.43, 2.5, 6.86])
def test_decode_schedule_spreads_the_cadence(ratio):
    sched = decode_schedule(30, ratio)
    assert len(sched) == 30 and min(sched) >= 1
    assert abs(sum(sched) - 30 * ratio) < 1.0 + 1e-9
    assert max(sched) - min(sched) <= 1
    assert decode_schedule(3, 2) == [2, 2, 2] and decode_schedule(2, [1, 3]) == [1, 3]
    with pytest.raises(ValueError):
        decode_schedule(2, [1])


def test_page_allocator_and_buckets():
    a = PageAllocator(10)
    got = a.alloc(4)
    assert 0 not in got and len(set(got)) == 4  # page 0 is the scratch page
    a.release(got)
    assert len(a.alloc(9)) == 9
    with pytest.raises(InvalidArgumentError):
        a.alloc(1)
    assert [bucket_of(b) for b in (1, 8, 9, 33, 256)] == [8, 8, 16, 64, 256]
    assert BUCKETS[-1] == 256
    with pytest.raises(InvalidArgumentError):
        bucket_of(257)


def test_kv_pages_cover_the_reference_admission_budget():
    cfg = E.SimConfig(gpu=b200_gpu(), model=M, slo=S.SloSpec(3e-3, 0.15))
    pages = kv_pages_for(cfg, max_live_requests=100)
    budget = cfg.kv_pool_bytes - M.weight_bytes()
    # any admitted set (sum of kv_bytes <= budget) fits in whole pages plus
    # one partial page per live request, plus the scratch page
    assert (pages - 100 - 1) * kv_bytes(M, 64) <= budget < (pages - 100) * kv_bytes(M, 64)


def test_decision_fixture_codecs_round_trip():
    rnd = random.Random(1)
    decisions, alpha = [], {}
    for i in range(30):
        alpha[("decode", rnd.choice([8, 16, 148]), rnd.randint(1, 9999))] = rnd.random()
        st = corun_state(4096, [rnd.randint(100, 4000) for _ in range(5)], 148, dm0=16)
        st.tpot_window = tuple(rnd.random() for _ in range(3))
        decisions.append({"kind": "decode", "state": state_to_json(st),
                          "store": {"alpha": [[*k, v] for k, v in alpha.items()],
                                    "contention": [[8, 1024, 1e12]]},
                          "decision": {"batch": [1, 2], "predicted_step_s": 0.1}})
    back = delta_decode(delta_encode(decisions))
    for a, b in zip(decisions, back):
        assert sorted(map(tuple, a["store"]["alpha"])) == sorted(map(tuple, b["store"]["alpha"]))
        s1 = state_from_json(a["state"], (S, PM))
        s2 = state_from_json(b["state"], (S, PM))
        assert s1.es == s2.es and s1.tpot_window == s2.tpot_window and s1.decode_running == s2.decode_running
        st = store_from_json(b["store"], PM)
        assert st.alpha_samples == {(k[0], k[1], k[2]): k[3] for k in a["store"]["alpha"]}


def test_incremental_store_axes_equal_a_rebuild():
    rnd = random.Random(7)
    inc, ref = PM.CalibrationStore(), PM.CalibrationStore()
    for i in range(2000):
        key = (rnd.choice(["prefill", "decode"]), rnd.choice([8, 16, 24, 140, 148]), rnd.randint(1, 3000))
        v = 0.5 + rnd.random()
        inc.alpha_for(key[0], 40, 100)  # keep the cache warm so set_alpha updates it in place
        inc.set_alpha(key, v)
        ref.alpha_samples[key] = v
        ref._invalidate()
        if i % 50 == 0:
            for ph in ("prefill", "decode"):
                assert inc._axes(ph) == ref._axes(ph)
                a, b = rnd.randint(1, 148), rnd.randint(1, 5000)
                assert inc.alpha_for(ph, a, b) == ref.alpha_for(ph, a, b)
