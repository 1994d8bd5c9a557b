"""The SM split of a co-executed prefill layer + decode step, chosen by the
reference's own estimator and scheduler functions (not by measurement).

Algorithm 1 (reference scheduler.py:311-372) in the
steady state of BASELINE config 2 -- one prefill request of T tokens in
flight, a decode batch running beside it:

  * "During concurrent operation, the decode phase is provisioned with the
    minimum SM counts that satisfy SLO": dm =
    `min_decode_sms` (scheduler.py:267-279) on the 8-SM green-context grid,
    with the decode step predicted under the co-running prefill's HBM
    contention (perf_model.py:386-414, the B200 calibration store);
  * if the prefill's projected TTFT then misses its target as well, both
    SLOs are violated and Algorithm 1 takes the balanced branch:
    `set_balanced_sm` (scheduler.py:241-264).

The estimator reads the tables re-measured on the B200 (profiles/calib_b200,
device/calibrate.py): alpha / contention samples and the measured n_d.
"""

from __future__ import annotations

import json
from pathlib import Path

from ..perf_model import CalibrationStore, ExecutionState, PerfEstimator, b200_spec
from ..scheduler import (PrefillState, ReqView, SchedulerConfig, SloSpec, SystemState, _prefill_ttft_ratio,
                         min_decode_sms, set_balanced_sm)

ROOT = Path(__file__).resolve().parents[2]
CALIB = ROOT / "profiles" / "calib_b200"


def b200_gpu(calib: Path = CALIB):
    """GpuSpec with the B200-measured peaks and n_d from the calibration run."""
    g = calib / "gpu.json"
    if g.exists():
        d = json.loads(g.read_text())
        return b200_spec(c_peak=d["c_peak"], d_peak=d["d_peak"], n_d=d["n_d"], n_w=d["n_w"])
    return b200_spec()


def b200_store(calib: Path = CALIB) -> CalibrationStore:
    """The B200-measured calibration store (reference JSONL format)."""
    p = calib / "calibration.jsonl"
    if not p.exists():
        raise FileNotFoundError(f"{p}: run device/calibrate.py on the B200 first")
    return CalibrationStore.load_jsonl(p)


def corun_state(T: int, ctx_lens, n: int, dm0: int = 8) -> SystemState:
    """SystemState of config 2: request 0 (T prompt tokens) in flight at
    layer 0, requests 1..B decoding with the given contexts."""
    reqs = {0: ReqView(0, 0.0, T, 0)}
    for i, c in enumerate(ctx_lens, start=1):
        reqs[i] = ReqView(i, 0.0, int(c), int(c))
    es = ExecutionState(prefill_lens=(T,), prefill_sms=n - dm0,
                        decode_ctx_lens=tuple(int(c) for c in ctx_lens), decode_sms=dm0)
    return SystemState(es=es, ps=PrefillState([], [0], 0), requests=reqs, sim_time=0.0,
                       decode_running=tuple(range(1, len(ctx_lens) + 1)))


def estimator_split(model, T: int, ctx_lens, slo: SloSpec, gpu=None, store: CalibrationStore | None = None,
                    sm_step: int = 8) -> dict:
    """(pm, dm) for config 2 from the reference's estimator + Algorithm 1
    (module docstring), with the predictions behind it.  `slo` is in the
    reference's whole-model units (normalised TTFT per prompt token; TPOT
    per whole-model decode step)."""
    gpu = gpu or b200_gpu()
    store = store if store is not None else b200_store()
    est = PerfEstimator(model, gpu, store)
    cfg = SchedulerConfig(sm_step=sm_step)
    n = gpu.num_sms
    state = corun_state(T, ctx_lens, n, dm0=sm_step)
    dm = min_decode_sms(state, slo, est, cfg)
    branch = "min_decode_sms"
    if dm >= n:  # no share meets the TPOT target: Algorithm 1's balanced branch
        dm = n - sm_step
    pm = n - dm
    r_prefill = _prefill_ttft_ratio(state, slo, est, pm, [])
    r_decode = est.decode_step_s(list(ctx_lens), dm, T) / slo.tpot_s
    if r_prefill > 1.0:
        pm, dm = set_balanced_sm(state, slo, est, cfg)
        branch = "set_balanced_sm"
        r_prefill = _prefill_ttft_ratio(state, slo, est, pm, [])
        r_decode = est.decode_step_s(list(ctx_lens), dm, T) / slo.tpot_s
    return {"pm": pm, "dm": dm, "branch": branch, "sm_step": sm_step,
            "predicted_prefill_layer_s": est.prefill_layer_s([T], pm),
            "predicted_decode_layer_s": est.decode_step_s(list(ctx_lens), dm, T) / model.num_layers,
            "ttft_ratio": r_prefill, "tpot_ratio": r_decode,
            "slo": {"norm_ttft_s_per_token": slo.norm_ttft_s_per_token, "tpot_s": slo.tpot_s}}
