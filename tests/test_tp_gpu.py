"""TPLayer (device/tp.py) on the B200 kernels: two ranks of a TP=2 split run
as two processes sharing cuda:0 (gloo carries the all-reduces, staged in
fp32), and their output must match the unsharded CPU oracle layer within the
bf16 tolerance of tests/parity_harness.py."""

import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from parity_harness import ATOL, excess  # noqa: E402

from oracle import numerics as O  # noqa: E402

H, HQ, HKV, D, INTER, T, B, CTX = 1024, 8, 2, 128, 2048, 300, 4, 200


def _bf(a):
    return O.bf16_round(np.asarray(a, np.float32))


def _weights():
    rng = np.random.default_rng(11)
    W = O.LayerWeights(_bf(rng.normal(0, 0.02, ((HQ + 2 * HKV) * D, H))), _bf(rng.normal(0, 0.02, (H, H))),
                       _bf(rng.normal(0, 0.02, (INTER, H))), _bf(rng.normal(0, 0.02, (INTER, H))),
                       _bf(rng.normal(0, 0.02, (H, INTER))), _bf(1 + 0.1 * rng.normal(size=H)),
                       _bf(1 + 0.1 * rng.normal(size=H)))
    return W, _bf(rng.normal(size=(T, H))), _bf(rng.normal(size=(B, H)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, fused=False):
    two_shot = fused == "two_shot"
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_19516_b200.device import lib
    from paper_2504_19516_b200.device.tp import TPLayer, shard_dense, tp_shape

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)

    def ar(t):  # fp32-staged host all-reduce (two ranks share one GPU)
        torch.cuda.current_stream().synchronize()
        c = t.float().cpu()
        dist.all_reduce(c)
        t.copy_(c.to(dev))

    W, x, xd = _weights()

    def tt(a, dt=torch.bfloat16):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

    parts = shard_dense(W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, HQ, HKV, D, rank, world)
    lyr = TPLayer(tp_shape(H, HQ, HKV, D, INTER, world), *[tt(p) for p in parts], tt(W.attn_norm),
                  tt(W.mlp_norm), rank, device=dev, max_tokens=T, max_pos=1024, allreduce=ar)
    if fused:  # decode all-reduces through the GEMM epilogue over CUDA IPC peer memory
        from paper_2504_19516_b200.device.peer import PeerAllReduce

        lyr.peer = PeerAllReduce.create(dist.group.WORLD, B, H, dev, two_shot=two_shot)
    kvh = HKV // world
    pages = -(-T // 64)
    kc = torch.zeros(pages + B * 4, kvh, 64, D, dtype=torch.bfloat16, device=dev)
    vc = torch.zeros_like(kc)
    y = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    lyr.prefill(tt(x), y, torch.tensor([0, T], **i32), 1, T, torch.arange(T, **i32), torch.arange(T, **i32),
                kc, vc, 148)
    torch.cuda.synchronize()
    # decode: B sequences with their own pages after the prefill's
    bt = (pages + torch.arange(B * 4, **i32)).view(B, 4)
    ctx = torch.full((B,), CTX, **i32)
    pos = ctx - 1
    slots = bt[torch.arange(B), pos // 64] * 64 + pos % 64
    ws = torch.empty(lib.decode_attn_ws_bytes(B, HQ // world, D, 64) // 4 + 1, dtype=torch.float32, device=dev)
    yd = torch.empty(B, H, dtype=torch.bfloat16, device=dev)
    lyr.decode(tt(xd), yd, ctx, pos, slots, bt, kc, vc, 148, ws=ws)
    torch.cuda.synchronize()
    if fused:
        yd2 = torch.empty_like(yd)  # second call: the other buffer half, epoch 3/4
        lyr.decode(tt(xd), yd2, ctx, pos, slots, bt, kc, vc, 148, ws=ws)
        torch.cuda.synchronize()
        assert torch.equal(yd, yd2)
        dist.barrier()
        lyr.peer.close()
    q.put((rank, y.float().cpu().numpy(), yd.float().cpu().numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [False, True, "two_shot"], ids=["nccl_style", "fused_peer", "fused_two_shot"])
def test_tp2_layer_on_device_matches_oracle(fused):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, fused)) for r in range(world)]
    for p in procs:
        p.daemon = True
        p.start()
    outs = {}
    try:
        for _ in range(world):
            r, y, yd = q.get(timeout=300)
            outs[r] = (y, yd)
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    W, x, xd = _weights()
    table = O.rope_table(1024, D)
    ref, _, _ = O.layer_prefill(x, W, HQ, HKV, D, np.arange(T), table, bf16_boundaries=True)
    assert np.array_equal(outs[0][0], outs[1][0])  # replicated after the all-reduce
    if fused:
        assert np.array_equal(outs[0][1], outs[1][1])
    assert excess(outs[0][0], ref) <= ATOL
    # decode oracle over the same cache contents: positions < CTX-1 of the decode
    # sequences were never written (zero K/V), exactly as on the device
    kc = np.zeros((-(-T // 64) + B * 4, HKV, 64, D), np.float32)
    vc = np.zeros_like(kc)
    bt = (-(-T // 64) + np.arange(B * 4)).reshape(B, 4)
    refd = O.layer_decode(xd, W, HQ, HKV, D, np.full(B, CTX), table, kc, vc, bt, bf16_boundaries=True)
    assert excess(outs[0][1], refd) <= ATOL
