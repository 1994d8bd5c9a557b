"""BASELINE config 4: Llama-3-8B serving on a synthetic Poisson trace, one
independent replica per GPU, with every step time measured on the B200.

Each rank takes the requests with id % world == rank (the path shards only
by request) and runs the reference's serving loop
(`engine.run`, reference engine.py:860-880) for each policy with the device
seam bound to `B200Executor`: prefill layers on pm-SM green contexts
co-executed with decode steps on dm SMs (bullet), the lockstep chunked-prefill
baseline on hybrid batches (chunked), and both phases on the whole GPU
(nopartition, time-sliced).  The estimator reads the calibration tables
re-measured on the B200 (profiles/calib_b200, device/calibrate.py) instead
of sampling the synthetic surfaces.

    python -m paper_2504_19516_b200.device.serve --rate 4 --duration 20
    torchrun --nproc-per-node 8 -m paper_2504_19516_b200.device.serve ...

Rank 0 prints one JSON line per policy: total tokens / max-over-ranks
makespan, and the replicas' p50 TTFT / TPOT (median over replicas).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
from pathlib import Path

from .. import engine as E
from .. import scheduler as S
from ..perf_model import CalibrationStore, b200_spec
from ..workload import MODEL_PRESETS, LengthDist, Request, TRACE_PRESETS, gen_poisson_trace

ROOT = Path(__file__).resolve().parents[2]
CALIB = ROOT / "profiles" / "calib_b200"


def b200_gpu():
    """GpuSpec with the B200-measured n_d / D from the calibration run."""
    g = CALIB / "gpu.json"
    if g.exists():
        d = json.loads(g.read_text())
        return b200_spec(c_peak=d["c_peak"], d_peak=d["d_peak"], n_d=d["n_d"], n_w=d["n_w"])
    return b200_spec()


def shard(trace, rank: int, world: int):
    """Requests of replica `rank` (id mod world), ids renumbered densely."""
    mine = [r for r in trace if r.id % world == rank]
    return [Request(i, r.arrival_s, r.input_len, r.output_len) for i, r in enumerate(mine)]


def run_policy(policy: str, trace, ex, gpu, chunk: int = 1024):
    model = MODEL_PRESETS["llama3-8b"]
    g = CALIB / "gpu.json"
    reconfig = json.loads(g.read_text()).get("reconfig_s") if g.exists() else None
    cfg = E.SimConfig(gpu=gpu, model=model,
                      slo=S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.1),
                      sched=S.SchedulerConfig(sm_step=8),
                      policy=E.PolicySpec(policy, chunk_size=chunk), seed=0,
                      **({"reconfig_s": reconfig} if reconfig is not None else {}))
    store = CalibrationStore.load_jsonl(CALIB / "calibration.jsonl") if (CALIB / "calibration.jsonl").exists() else None
    rep = E.run(cfg, trace, oracle=ex, store=store)
    a = dict(rep.aggregates)
    a.update(rep.extended)
    return a


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=4.0, help="requests/s (whole job)")
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policies", default="bullet,chunked,nopartition")
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--out", default=None)
    ap.add_argument("--full-model", action="store_true",
                    help="keep all 32 layers resident: decode steps measured over the whole model, "
                         "prefill steps over l_step distinct layers")
    a = ap.parse_args(argv)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # control plane only: JSON results

    from .executor import B200Executor

    gpu = b200_gpu()
    # config 4 prompt lengths: uniform 512-8192; outputs from the ShareGPT-like preset
    trace = gen_poisson_trace(a.rate, a.duration, LengthDist("uniform", lo=512, hi=8192),
                              TRACE_PRESETS["sharegpt-like"][1], seed=a.seed)
    mine = shard(trace, rank, world)
    ex = B200Executor(MODEL_PRESETS["llama3-8b"], gpu, device=local, max_prefill_tokens=65536,
                      max_decode_batch=256, pool_tokens=(1 << 18) if a.full_model else (1 << 20), memo=True,
                      full_model=a.full_model)
    lines = []
    for pol in a.policies.split(","):
        agg = run_policy(pol, mine, ex, gpu, a.chunk)
        per = [agg]
        if dist is not None:
            per = [None] * world
            dist.all_gather_object(per, agg)
        if rank == 0:
            span = max(p["makespan_s"] for p in per)
            toks = sum(p.get("tokens_finished", 0) for p in per)
            line = {"config": "llama3-8b serving, Poisson trace, prompts U[512,8192]", "policy": pol,
                    "replicas": world, "rate_rps": a.rate, "duration_s": a.duration,
                    "requests": len(trace), "finished": sum(p["finished"] for p in per),
                    "tokens_per_s": toks / span if span > 0 else 0.0, "makespan_s": span,
                    "p50_ttft_s": statistics.median(p.get("ttft_p50_s", 0.0) for p in per),
                    "p50_tpot_ms": statistics.median(p.get("tpot_p50_ms", 0.0) for p in per),
                    "p90_tpot_ms": statistics.median(p["tpot_p90_ms"] for p in per),
                    "slo_attainment": statistics.mean(p["slo_attainment"] for p in per),
                    "mean_prefill_sms": statistics.mean(p["mean_prefill_sms"] for p in per),
                    "mean_decode_sms": statistics.mean(p["mean_decode_sms"] for p in per),
                    "device_calls": dict(ex.calls), "memo_hits": ex.memo_hits,
                    "timing": "every step time measured on the B200 (CUDA events, green-context partitions)",
                    "measured_unit": "whole-model decode step, l_step prefill layers" if a.full_model
                    else "one resident layer x num_layers"}
            print(json.dumps(line), flush=True)
            lines.append(line)
    if rank == 0 and a.out:
        Path(a.out).write_text("\n".join(json.dumps(x) for x in lines) + "\n")
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
