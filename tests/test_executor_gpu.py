"""B200Executor: the reference's oracle protocol backed by measured kernels,
driving the reference event loop (engine.run(..., oracle=...))."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_19516_b200 import engine as E  # noqa: E402
from paper_2504_19516_b200 import scheduler as S  # noqa: E402
from paper_2504_19516_b200.perf_model import ExecutionState, b200_spec, srm_prefill_layer_s  # noqa: E402
from paper_2504_19516_b200.workload import MODEL_PRESETS, Request  # noqa: E402


@pytest.fixture(scope="module")
def ex():
    from paper_2504_19516_b200.device.executor import B200Executor

    return B200Executor(MODEL_PRESETS["llama3-8b"], b200_spec(), max_prefill_tokens=8192,
                        max_decode_batch=64, pool_tokens=1 << 18)


def test_measured_prefill_layer_is_plausible(ex):
    m = MODEL_PRESETS["llama3-8b"]
    es = ExecutionState(prefill_lens=(2048,), prefill_sms=148)
    t = ex.prefill_layer_s(es)
    srm = srm_prefill_layer_s(es, m, b200_spec())
    assert 0.8 * srm < t < 4.0 * srm, (t, srm)
    # fewer SMs -> slower
    t_small = ex.prefill_layer_s(ExecutionState(prefill_lens=(2048,), prefill_sms=84))
    assert t_small > t


def test_measured_decode_step_and_contention(ex):
    es = ExecutionState(decode_ctx_lens=(1024,) * 16, decode_sms=32)
    alone = ex.decode_step_s(es)
    co = ex.decode_step_s(ExecutionState(prefill_lens=(4096,), prefill_sms=116,
                                         decode_ctx_lens=(1024,) * 16, decode_sms=32))
    assert alone > 0 and co > 0
    assert ex.contention_bw(32, 0) > 1e12
    assert 0.1 < ex.alpha("prefill", 148, 2048) < 10


def test_engine_runs_on_measured_latencies(ex):
    gpu = b200_spec()
    cfg = E.SimConfig(gpu=gpu, model=MODEL_PRESETS["llama3-8b"],
                      slo=S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.1),
                      sched=S.SchedulerConfig(sm_step=8), seed=0)
    trace = [Request(i, 0.002 * i, 512 + 256 * i, 4) for i in range(6)]
    rep = E.run(cfg, trace, oracle=ex)
    assert rep.aggregates["finished"] == len(trace)
    for entry in rep.decision_log:
        assert entry["dm"] % 8 == 0 or entry["dm"] == gpu.num_sms
    assert ex.calls["prefill"] > 0 and ex.calls["decode"] > 0


def test_hybrid_iteration_and_chunked_policy_on_hardware(ex):
    # GroundTruthOracle.hybrid_iteration_s (engine.py:200-208) measured on the B200
    t1 = ex.hybrid_iteration_s([(1024, 0)], [], 148)
    t2 = ex.hybrid_iteration_s([(1024, 3072)], [2048] * 32, 148)
    t3 = ex.hybrid_iteration_s([], [1024] * 16, 148)
    assert 0 < t3 < t1 < t2
    gpu = b200_spec()
    cfg = E.SimConfig(gpu=gpu, model=MODEL_PRESETS["llama3-8b"],
                      slo=S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.1),
                      policy=E.PolicySpec(name="chunked", chunk_size=1024), seed=0)
    trace = [Request(i, 0.002 * i, 512 + 256 * i, 4) for i in range(6)]
    rep = E.run(cfg, trace, oracle=ex)
    assert rep.aggregates["finished"] == len(trace)
    assert ex.calls["hybrid"] > 0


def test_full_model_executor_measures_whole_decode_step():
    # every layer resident, decode measured over the whole model
    from paper_2504_19516_b200.device.executor import B200Executor

    m = MODEL_PRESETS["llama3-8b"]
    fx = B200Executor(m, b200_spec(), max_prefill_tokens=4096, max_decode_batch=32, pool_tokens=1 << 15,
                      full_model=True, l_step=4)
    assert len(fx.layers) == m.num_layers and fx.l_step == 4
    es = ExecutionState(decode_ctx_lens=(1024,) * 16, decode_sms=148)
    step = fx.decode_step_s(es)
    pl = fx.prefill_layer_s(ExecutionState(prefill_lens=(2048,), prefill_sms=148))
    assert 0 < pl < 0.01 and 32 * 40e-6 < step < 0.1
    del fx
    torch.cuda.empty_cache()
