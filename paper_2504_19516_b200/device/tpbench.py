"""BASELINE config 5: Llama-3-70B layer, tensor parallel, chunked prefill
2048 + decode batch 128 (ctx 2048), one process per GPU.

    torchrun --nproc-per-node 8 -m paper_2504_19516_b200.device.tpbench
    python -m paper_2504_19516_b200.device.tpbench --tp 8     # 1 GPU: rank-0 shard, no collective

Each phase gets its own NCCL communicator and its
all-reduces run on the phase's stream, so on a green-context split they are
charged to that phase's SMs.  Rank 0 prints one JSON line: per-layer
prefill / decode times alone and co-run on (pm, dm), and the all-reduce
bytes per layer (2 x T x hidden x 2 B).
"""

from __future__ import annotations

import argparse
import json
import os

import torch

from ..workload import MODEL_PRESETS
from . import lib
from .partition import DECODE, PREFILL, PartitionPool
from .tp import TPLayer, tp_shape


def _ev():
    return torch.cuda.Event(enable_timing=True)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=None, help="shard shapes for this TP degree (default WORLD_SIZE)")
    ap.add_argument("--prefill", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--dm", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fused", action="store_true",
                    help="decode all-reduces fused into the o_proj/mlp_down epilogues (device/peer.py); on 1 GPU "
                         "the tp ranks' receive buffers are emulated locally and peers' flags pre-raised")
    ap.add_argument("--two-shot", action="store_true", help="with --fused: reduce-scatter + all-gather form")
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    tp = a.tp or world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    groups = (None, None)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        groups = (dist.new_group(list(range(world))), dist.new_group(list(range(world))))
    m = MODEL_PRESETS["llama3-70b"]
    s = tp_shape(m.hidden, m.num_heads, m.num_kv_heads, m.head_dim, m.intermediate, tp)
    g = torch.Generator(device="cpu").manual_seed(rank)

    def w(*shape):
        return (torch.randn(*shape, generator=g) * 0.02).to(torch.bfloat16).to(dev)

    nrm = torch.ones(m.hidden, dtype=torch.bfloat16, device=dev)
    args = (w(s.qkv_out, s.hidden), w(s.hidden, s.heads * s.head_dim), w(s.inter, s.hidden), w(s.inter, s.hidden),
            w(s.hidden, s.inter), nrm, nrm)
    T, B, C = a.prefill, a.batch, a.ctx
    pl = TPLayer(s, *args, rank, group=groups[0], device=dev, max_tokens=T, max_pos=max(T, C) + 1)
    dl = TPLayer(s, *args, rank, group=groups[1], device=dev, max_tokens=B, max_pos=max(T, C) + 1)
    if a.fused:
        from .peer import PeerAllReduce

        if world > 1:
            dl.peer = PeerAllReduce.create(groups[1], B, s.hidden, dev, device_epoch=True, two_shot=a.two_shot)
        else:  # rank 0's view of a tp-rank group: scatter to tp local buffers, peers' flags pre-raised
            dl.peer = PeerAllReduce.local_group(tp, B, s.hidden, dev, device_epoch=True, two_shot=a.two_shot)[0]
            dl.peer.flags.fill_(2 ** 31 - 1)
            if a.two_shot:
                dl.peer.gather[1].fill_(2 ** 31 - 1)
    bf = dict(dtype=torch.bfloat16, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    px, py = torch.randn(T, s.hidden, **bf), torch.empty(T, s.hidden, **bf)
    dx, dy = torch.randn(B, s.hidden, **bf), torch.empty(B, s.hidden, **bf)
    pages = -(-C // 64)
    nblk = -(-T // 64) + B * pages
    kc = torch.randn(nblk, s.kv_heads, 64, s.head_dim, **bf)
    vc = torch.randn_like(kc)
    cu = torch.tensor([0, T], **i32)
    ppos = torch.arange(T, **i32)
    bt = (-(-T // 64) + torch.arange(B * pages, **i32)).view(B, pages)
    ctx = torch.full((B,), C, **i32)
    dpos = ctx - 1
    dslots = bt[torch.arange(B, device=dev), dpos // 64] * 64 + dpos % 64
    ws = torch.empty(lib.decode_attn_ws_bytes(B, s.heads, s.head_dim, 4 * pages + 8) // 4 + 1,
                     dtype=torch.float32, device=dev)
    pool = PartitionPool(local)

    def run_p(st):
        pl.prefill(px, py, cu, 1, T, ppos, ppos, kc, vc, st.sms, st.torch_stream)

    graphs = {}

    def run_d(st):
        """One decode layer-step, replayed from a CUDA graph captured on the
        phase's stream (eager launches of ~12 kernels are host-bound; the
        fused all-reduce uses device epochs so its graph replays)."""
        key = (st.stream, st.sms)
        if key not in graphs:
            with torch.cuda.stream(st.torch_stream):
                dl.decode(dx, dy, ctx, dpos, dslots, bt, kc, vc, st.sms, st.torch_stream, ws=ws)  # warm
                st.torch_stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st.torch_stream):
                    dl.decode(dx, dy, ctx, dpos, dslots, bt, kc, vc, st.sms, st.torch_stream, ws=ws)
            torch.cuda.synchronize()
            graphs[key] = g
        graphs[key].replay()

    def timed(fn, st):
        with torch.cuda.stream(st.torch_stream):
            fn(st)
            torch.cuda.synchronize()
            evs = []
            for _ in range(a.reps):
                e0, e1 = _ev(), _ev()
                e0.record(st.torch_stream)
                fn(st)
                e1.record(st.torch_stream)
                evs.append((e0, e1))
        torch.cuda.synchronize()
        return sorted(x.elapsed_time(y) for x, y in evs)[len(evs) // 2] * 1e3

    full = pool.full(PREFILL)
    t_p = timed(run_p, full)
    t_d = timed(run_d, pool.full(DECODE))
    ps, ds = pool.split(pool.n - a.dm, a.dm)
    # co-run: prefill layers on pm SMs while decode layers stream on dm SMs
    start, ep, ed = _ev(), _ev(), _ev()
    torch.cuda.synchronize()
    start.record()
    ps.torch_stream.wait_event(start)
    ds.torch_stream.wait_event(start)
    with torch.cuda.stream(ps.torch_stream):
        for _ in range(a.reps):
            run_p(ps)
        ep.record(ps.torch_stream)
    with torch.cuda.stream(ds.torch_stream):
        for _ in range(a.reps * 4):
            run_d(ds)
        ed.record(ds.torch_stream)
    torch.cuda.synchronize()
    co_p = start.elapsed_time(ep) * 1e3 / a.reps
    co_d = start.elapsed_time(ed) * 1e3 / (4 * a.reps)
    if rank == 0:
        print(json.dumps({
            "config": f"llama3-70b layer TP={tp}: chunked prefill {T} + decode batch {B} ctx {C}",
            "world": world,
            "collective": (f"decode: fused GEMM-epilogue peer all-reduce ({'two' if a.two_shot else 'one'}-shot) x2 "
                           "per layer; prefill: " if a.fused else "")
            + ("nccl all-reduce x2 per layer" if world > 1 else
               "none (1 GPU: rank-0 shard compute only" + (", fused epilogue scatter to tp local buffers)"
                                                           if a.fused else ")")),
            "prefill_layer_us": t_p, "decode_layer_us": t_d,
            "corun": {"pm": pool.n - a.dm, "dm": a.dm, "prefill_layer_us": co_p, "decode_layer_us": co_d},
            "allreduce_bytes_per_layer": {"prefill": 2 * T * s.hidden * 2, "decode": 2 * B * s.hidden * 2},
            "local_shapes": {"qkv_out": s.qkv_out, "heads": s.heads, "kv_heads": s.kv_heads, "inter": s.inter},
        }), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
