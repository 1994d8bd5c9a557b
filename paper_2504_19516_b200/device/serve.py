"""BASELINE config 4: Llama-3-8B serving on a synthetic Poisson trace, one
independent replica per GPU, with the device doing the work.

Each rank takes the requests with id % world == rank (the path shards only
by request) and serves them with three policies:
bullet (the reference's Algorithm 1, prefill layers on pm-SM green contexts
co-executed with decode steps on dm SMs), chunked (lockstep hybrid batches,
SGLang-style) and nopartition (both phases on the whole GPU, time-sliced by
the hardware).  Two modes:

  --realtime   (default)  device/realtime.py: the reference's event loop on a
               wall clock; all 32 layers resident, real tokens generated,
               every decode step ONE CUDA graph (embedding .. LM head +
               argmax) replayed on the decode partition, completion events
               feeding update_online / the TPOT window.  Throughput and
               latencies are wall-clock and include the Python control
               plane.
  --replay     the reference's simulated clock with every step time
               measured on the device (device/executor.py B200Executor,
               optionally memoised) -- the round-1 mode, kept for
               comparison with the reference simulator.

    python -m paper_2504_19516_b200.device.serve --rate 4 --duration 10
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
from ..perf_model import CalibrationStore
from ..workload import MODEL_PRESETS, LengthDist, Request, TRACE_PRESETS, gen_poisson_trace
from .split import CALIB, b200_gpu

ROOT = Path(__file__).resolve().parents[2]
VOCAB = 128256  # Llama-3 tokenizer size (random-init embedding / LM head)
# PAPER.md:690-705 Table "Workload latency requirements", ShareGPT column
PAPER_SLO = S.SloSpec(norm_ttft_s_per_token=3.0e-3, tpot_s=0.150)


def shard(trace, rank: int, world: int):
    """Requests of replica `rank` (id mod world), ids renumbered densely."""
    mine = [r for r in trace if r.id % world == rank]
    return [Request(i, r.arrival_s, r.input_len, r.output_len) for i, r in enumerate(mine)]


def sim_config(policy: str, gpu, slo: S.SloSpec, chunk: int = 1024, realtime: bool = True,
               static_pm: int = 116) -> E.SimConfig:
    model = MODEL_PRESETS["llama3-8b"]
    g = CALIB / "gpu.json"
    reconfig = json.loads(g.read_text()).get("reconfig_s") if g.exists() else None
    kw = {"reconfig_s": reconfig} if reconfig is not None else {}
    if realtime:  # the control plane's cost is real, not modelled
        kw.update(metadata_overhead_s=0.0, predict_overhead_s=0.0)
    return E.SimConfig(gpu=gpu, model=model, slo=slo, sched=S.SchedulerConfig(sm_step=8),
                       policy=E.PolicySpec(policy, chunk_size=chunk, static_pm=static_pm), seed=0, **kw)


def calib_store():
    p = CALIB / "calibration.jsonl"
    return CalibrationStore.load_jsonl(p) if p.exists() else None


def run_replay(policy: str, trace, ex, gpu, slo, chunk: int):
    rep = E.run(sim_config(policy, gpu, slo, chunk, realtime=False), trace, oracle=ex, store=calib_store())
    a = dict(rep.aggregates)
    a.update(rep.extended)
    return a


def run_realtime(policy: str, trace, server, pool, gpu, slo, chunk: int, decisions_out=None, max_decisions=400,
                 static_pm: int = 116):
    from .realtime import RealtimeChunked, RealtimeSim, delta_encode

    serialize = policy == "timesliced"  # nopartition with both phases on one stream
    cfg = sim_config("nopartition" if serialize else policy, gpu, slo, chunk, static_pm=static_pm)
    if policy == "chunked":
        sim = RealtimeChunked(cfg, trace, server, pool)
    else:
        sim = RealtimeSim(cfg, trace, server, pool, store=calib_store(), trace_decisions=decisions_out is not None,
                          serialize=serialize)
    rep = sim.run()
    a = dict(rep.aggregates)
    a.update(rep.extended)
    a.update(wall_s=sim.wall_s, host_busy_s=sim.host_busy_s, control_plane_frac=sim.host_busy_s / sim.wall_s,
             device_calls=dict(sim.device_calls),
             step_gap_us={ph: (1e6 * statistics.mean(v) if v else None) for ph, v in getattr(sim, "gaps", {}).items()},
             generated_tokens=sum(len(v) for v in sim.generated.values()))
    if decisions_out is not None and policy == "bullet":
        g = gpu
        Path(decisions_out).write_text(json.dumps({
            "config": {"model": "llama3-8b", "slo": [slo.norm_ttft_s_per_token, slo.tpot_s], "sm_step": 8,
                       "l_step": cfg.sched.l_step, "num_sms": g.num_sms,
                       "gpu": {"name": g.name, "num_sms": g.num_sms, "c_peak": g.c_peak, "d_peak": g.d_peak,
                               "w_peak": g.w_peak, "n_d": g.n_d, "n_w": g.n_w}},
            "decisions": delta_encode(_spread(sim.decisions, max_decisions))}))
    return a


def _spread(xs, k):
    """At most k entries, evenly spread over the run (fixture size bound)."""
    if len(xs) <= k:
        return xs
    step = len(xs) / k
    return [xs[int(i * step)] for i in range(k)]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rate", type=float, default=4.0, help="requests/s (whole job)")
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policies", default="bullet,chunked,nopartition,timesliced",
                    help="timesliced = nopartition with both phases serialised on one stream (real time only)")
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--out", default=None)
    ap.add_argument("--replay", action="store_true", help="round-1 mode: simulated clock, measured step times")
    ap.add_argument("--full-model", action="store_true", help="(--replay) all 32 layers resident")
    ap.add_argument("--slo", default="paper", choices=["paper", "r01"],
                    help="paper: ShareGPT SLOs of PAPER.md Table (3.0 ms/token, 150 ms); r01: 1.5 ms, 100 ms")
    ap.add_argument("--static-pm", type=int, default=116,
                    help="policy static: fixed prefill share (decode gets the rest while prefill runs)")
    ap.add_argument("--slo-ms", default=None, help="norm_ttft_ms_per_token,tpot_ms (overrides --slo)")
    ap.add_argument("--decisions-out", default=None, help="(realtime bullet) log decisions for the replay test")
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

    gpu = b200_gpu()
    slo = PAPER_SLO if a.slo == "paper" else S.SloSpec(norm_ttft_s_per_token=1.5e-3, tpot_s=0.1)
    if a.slo_ms:
        p_ms, d_ms = (float(v) for v in a.slo_ms.split(","))
        slo = S.SloSpec(norm_ttft_s_per_token=p_ms * 1e-3, tpot_s=d_ms * 1e-3)
    # config 4 prompt lengths: uniform 512-8192; outputs from the ShareGPT-like preset
    out_dist = TRACE_PRESETS["sharegpt-like"][1]
    trace = gen_poisson_trace(a.rate, a.duration, LengthDist("uniform", lo=512, hi=8192), out_dist, seed=a.seed)
    mine = shard(trace, rank, world)
    model = MODEL_PRESETS["llama3-8b"]
    if a.replay:
        from .executor import B200Executor

        dev_obj = B200Executor(model, gpu, device=local, max_prefill_tokens=65536, max_decode_batch=256,
                               pool_tokens=(1 << 18) if a.full_model else (1 << 20), memo=True,
                               full_model=a.full_model)
    else:
        from .layer import PAGE
        from .partition import PartitionPool
        from .realtime import ServingModel, kv_pages_for

        pool = PartitionPool(local)
        pool.warm()
        cfg0 = sim_config("bullet", gpu, slo)
        server = ServingModel(model, VOCAB, torch.device("cuda", local), kv_pages=kv_pages_for(cfg0),
                              # the reference's _form_batch has no token cap (static /
                              # nopartition batch a long queue at once): 192k packed tokens
                              max_prefill_tokens=196608, max_pages_per_seq=-(-(8192 + out_dist.hi + 1) // PAGE),
                              seed=a.seed + rank)
        graphs = server.warm(pool)
    lines = []
    for pol in a.policies.split(","):
        if a.replay:
            agg = run_replay(pol, mine, dev_obj, gpu, slo, a.chunk)
        else:
            agg = run_realtime(pol, mine, server, pool, gpu, slo, a.chunk,
                               a.decisions_out if rank == 0 else None, static_pm=a.static_pm)
        per = [agg]
        if dist is not None:
            per = [None] * world
            dist.all_gather_object(per, agg)
        if rank == 0:
            span = max(p["makespan_s"] for p in per)
            toks = sum(p.get("tokens_finished", 0) for p in per)
            line = {"config": "llama3-8b serving, Poisson trace, prompts U[512,8192]", "policy": pol,
                    "mode": "replay" if a.replay else "realtime", "replicas": world, "rate_rps": a.rate,
                    "duration_s": a.duration, "requests": len(trace), "finished": sum(p["finished"] for p in per),
                    "tokens_per_s": toks / span if span > 0 else 0.0, "makespan_s": span,
                    "p50_ttft_s": statistics.median(p.get("ttft_p50_s", 0.0) for p in per),
                    "p50_tpot_ms": statistics.median(p.get("tpot_p50_ms", 0.0) for p in per),
                    "p90_tpot_ms": statistics.median(p["tpot_p90_ms"] for p in per),
                    "mean_ttft_s": statistics.median(p["ttft_mean_s"] for p in per),
                    "slo_attainment": statistics.mean(p["slo_attainment"] for p in per),
                    "slo": {"norm_ttft_ms_per_token": 1e3 * slo.norm_ttft_s_per_token, "tpot_ms": 1e3 * slo.tpot_s},
                    "mean_prefill_sms": statistics.mean(p["mean_prefill_sms"] for p in per),
                    "mean_decode_sms": statistics.mean(p["mean_decode_sms"] for p in per)}
            if a.replay:
                line.update(device_calls=dict(dev_obj.calls), memo_hits=dev_obj.memo_hits,
                            timing="simulated clock; every step time measured on the B200")
            else:
                line.update(wall_s=max(p["wall_s"] for p in per),
                            control_plane_frac=statistics.mean(p["control_plane_frac"] for p in per),
                            device_calls=per[0]["device_calls"], decode_graphs_captured=graphs,
                            step_gap_us=per[0]["step_gap_us"],
                            generated_tokens=sum(p["generated_tokens"] for p in per),
                            timing="wall clock; real tokens; device completions from CUDA events")
            print(json.dumps(line), flush=True)
            lines.append(line)
    if rank == 0 and a.out:
        Path(a.out).write_text("\n".join(json.dumps(x) for x in lines) + "\n")
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
