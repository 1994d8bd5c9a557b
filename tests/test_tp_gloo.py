"""Tensor-parallel layer split (device/tp.py, BASELINE config 5) checked on
CPU with world_size 2 over gloo: each rank runs its Megatron shard (column-
parallel qkv / up-gate, row-parallel o_proj / down with the residual folded
in on rank 0) in the numpy oracle, the two all-reduces go through
torch.distributed, and the result must equal the unsharded oracle layer."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numerics as O
from paper_2504_19516_b200.device.tp import shard_dense, tp_shape


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(seed=0, h=64, Hq=4, Hkv=2, d=16, inter=96):
    rng = np.random.default_rng(seed)

    def w(*s):
        return (rng.normal(size=s) * 0.05).astype(np.float32)

    W = O.LayerWeights(w((Hq + 2 * Hkv) * d, h), w(h, h), w(inter, h), w(inter, h), w(h, inter),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32))
    x = rng.normal(size=(37, h)).astype(np.float32)
    return W, x, (h, Hq, Hkv, d, inter)


def _allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    dist.all_reduce(t)
    return t.numpy()


def _rank_main(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    W, x, (h, Hq, Hkv, d, inter) = _weights()
    s = tp_shape(h, Hq, Hkv, d, inter, world)
    wq, wo, wg, wu, wd = shard_dense(W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, Hq, Hkv, d, rank, world)
    T = x.shape[0]
    table = O.rope_table(64, d)
    pos = np.arange(T)
    qkv = O.rmsnorm(x, W.attn_norm) @ wq.T
    qq = O.apply_rope(qkv[:, :s.heads * d].reshape(T, s.heads, d), pos, table)
    kk = O.apply_rope(qkv[:, s.heads * d:(s.heads + s.kv_heads) * d].reshape(T, s.kv_heads, d), pos, table)
    vv = qkv[:, (s.heads + s.kv_heads) * d:].reshape(T, s.kv_heads, d)
    a = O.causal_attention(qq, kk, vv, 1.0 / math.sqrt(d)).reshape(T, s.heads * d)
    hh = _allreduce(a @ wo.T + (x if rank == 0 else 0.0))
    n2 = O.rmsnorm(hh, W.mlp_norm)
    act = O.silu(n2 @ wg.T) * (n2 @ wu.T)
    y = _allreduce(act @ wd.T + (hh if rank == 0 else 0.0))
    q.put((rank, y))
    dist.destroy_process_group()


def test_tp2_layer_equals_unsharded_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W, x, (h, Hq, Hkv, d, inter) = _weights()
    ref, _, _ = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(x.shape[0]), O.rope_table(64, d),
                                bf16_boundaries=False)
    for r in range(world):
        np.testing.assert_allclose(outs[r], ref, atol=2e-5, rtol=1e-4)


def test_shard_dense_partitions_every_weight_row_and_column():
    W, _, (h, Hq, Hkv, d, inter) = _weights()
    parts = [shard_dense(W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, Hq, Hkv, d, r, 2) for r in range(2)]
    assert sum(p[0].shape[0] for p in parts) == W.w_qkv.shape[0]
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts], axis=1), W.w_o)
    np.testing.assert_array_equal(np.concatenate([p[4] for p in parts], axis=1), W.w_down)
    with pytest.raises(ValueError):
        tp_shape(h, Hq, 3, d, inter, 2)
