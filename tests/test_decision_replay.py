"""Hardware decision replay (SURVEY 7 "Determinism", VERDICT r01 missing #6):
the real-time B200 engine (device/realtime.py, trace_decisions=True) logged
every scheduling call's exact SystemState, a snapshot of the calibration
store it held at that moment (alpha samples updated online from CUDA-event
measurements) and the decision it applied.  Here the REFERENCE's own
scheduler (/root/reference/pkg/src/smshare, when present) and this
package's scheduler are re-run on those logged inputs and must reproduce
every decision exactly: (pm, dm), branch, batch membership and order,
layers to run, and the decode step's predicted latency (IEEE-equal).

Fixtures: tests/golden/realtime_decisions_*.json, written by
tests/test_realtime_gpu.py (HP_DECISIONS_OUT) and
`python -m paper_2504_19516_b200.device.serve --decisions-out` (real-time mode)
on the B200.
"""

import contextlib
import importlib
import json
import sys
from pathlib import Path

import pytest

from paper_2504_19516_b200 import perf_model as PM
from paper_2504_19516_b200 import scheduler as S
from paper_2504_19516_b200 import workload as W
from paper_2504_19516_b200.device.realtime import delta_decode, state_from_json, store_from_json

GOLDEN = Path(__file__).resolve().parent / "golden"
FIXTURES = sorted(GOLDEN.glob("realtime_decisions_*.json"))
REF_SRC = Path("/root/reference/pkg/src")


@contextlib.contextmanager
def _reference():
    """smshare imported from the read-only reference tree (not the shim),
    live in sys.modules while the replay runs (its perf_model imports
    workload lazily at call time)."""
    if not (REF_SRC / "smshare").exists():
        pytest.skip("reference tree not present (GPU box)")
    saved = {k: sys.modules.pop(k) for k in list(sys.modules) if k == "smshare" or k.startswith("smshare.")}
    sys.path.insert(0, str(REF_SRC))
    try:
        sched = importlib.import_module("smshare.scheduler")
        pm = importlib.import_module("smshare.perf_model")
        wl = importlib.import_module("smshare.workload")
        assert Path(sched.__file__).resolve().is_relative_to(REF_SRC.resolve()), sched.__file__
        yield sched, pm, wl
    finally:
        sys.path.remove(str(REF_SRC))
        for k in [k for k in sys.modules if k == "smshare" or k.startswith("smshare.")]:
            sys.modules.pop(k)
        sys.modules.update(saved)


def _replay(fix, sched, pm, wl):
    cfgd = fix["config"]
    if cfgd["model"] == "tiny":
        t = W.TINY_MODEL
        model = wl.ModelSpec(t.name, num_layers=t.num_layers, hidden=t.hidden, num_heads=t.num_heads,
                             num_kv_heads=t.num_kv_heads, head_dim=t.head_dim, intermediate=t.intermediate)
    else:
        model = wl.MODEL_PRESETS[cfgd["model"]]
    gpu = pm.GpuSpec(**cfgd["gpu"])
    slo = sched.SloSpec(norm_ttft_s_per_token=cfgd["slo"][0], tpot_s=cfgd["slo"][1])
    scfg = sched.SchedulerConfig(sm_step=cfgd["sm_step"], l_step=cfgd["l_step"])
    L = model.num_layers
    counts = {"prefill": 0, "decode": 0, "branches": set()}
    for i, d in enumerate(delta_decode(fix["decisions"])):
        st = state_from_json(d["state"], (sched, pm))
        est = pm.PerfEstimator(model, gpu, store_from_json(d["store"], pm))
        if d["kind"] == "decode":
            got = sched.schedule_decode(st, slo, est, scfg)
            assert list(got.next_tasks) == d["decision"]["batch"], i
            assert got.predicted_step_s == d["decision"]["predicted_step_s"], i
        else:
            handoff = (st.ps.in_flight and not st.ps.queue and scfg.transition_layers > 0
                       and st.ps.layers_done >= L - scfg.transition_layers
                       and (st.decode_running or st.decode_ready))
            got = (sched.transition_handoff(st, scfg, gpu.num_sms, L) if handoff
                   else sched.schedule_prefill(st, slo, est, scfg))
            want = d["decision"]
            assert (got.new_prefill_sms, got.new_decode_sms, got.branch, list(got.next_tasks),
                    got.layers_to_run) == (want["pm"], want["dm"], want["branch"], want["batch"],
                                           want["layers"]), (i, want)
            counts["branches"].add(got.branch)
        counts[d["kind"]] += 1
    return counts


@pytest.mark.parametrize("fixture", FIXTURES, ids=[f.stem for f in FIXTURES])
def test_logged_b200_decisions_replay_with_this_package(fixture):
    fix = json.loads(fixture.read_text())
    c = _replay(fix, S, PM, W)
    assert c["prefill"] + c["decode"] == len(fix["decisions"]) > 0


@pytest.mark.parametrize("fixture", FIXTURES, ids=[f.stem for f in FIXTURES])
def test_logged_b200_decisions_replay_with_the_reference(fixture):
    fix = json.loads(fixture.read_text())
    with _reference() as (sched, pm, wl):
        c = _replay(fix, sched, pm, wl)
    assert c["prefill"] + c["decode"] == len(fix["decisions"]) > 0


def test_fixtures_exist():
    assert FIXTURES, "no logged B200 decision fixtures under tests/golden"
