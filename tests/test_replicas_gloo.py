"""Multi-replica plumbing on CPU (world_size 2, gloo): bench.py's split
agreement and whole-job totals (max-over-ranks span, summed tokens), and
serve.py's request sharding -- the N>1 paths the GPU box can only run with
one GPU."""

import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_2504_19516_b200.device.serve import shard
from paper_2504_19516_b200.workload import LengthDist, TRACE_PRESETS, gen_poisson_trace


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    split = tuple(bench.bcast(dist, [8 * (rank + 1), 1.5 + rank], "cpu"))
    span, tokens = bench.job_totals(dist, 0.010 + 0.005 * rank, 4128 * (rank + 1), "cpu")
    q.put((rank, split, span, tokens))
    dist.destroy_process_group()


def test_bench_job_totals_and_split_agreement_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, split, span, tokens in got:
        assert split == (8.0, 1.5)              # rank 0's decision everywhere
        assert abs(span - 0.015) < 1e-12        # max over ranks
        assert tokens == 4128 * 3               # whole-job tokens


def test_serve_shards_partition_the_trace():
    trace = gen_poisson_trace(8.0, 5.0, LengthDist("uniform", lo=512, hi=8192),
                              TRACE_PRESETS["sharegpt-like"][1], seed=3)
    parts = [shard(trace, r, 4) for r in range(4)]
    assert sum(len(p) for p in parts) == len(trace)
    for p in parts:
        assert [r.id for r in p] == list(range(len(p)))
        assert all(a.arrival_s <= b.arrival_s for a, b in zip(p, p[1:]))
    lens = sorted((r.input_len, r.output_len, r.arrival_s) for p in parts for r in p)
    assert lens == sorted((r.input_len, r.output_len, r.arrival_s) for r in trace)
