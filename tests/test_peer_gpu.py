"""Fused row-parallel GEMM + all-reduce (device/peer.py, include/hp.h
hp_gemm_swap_peer / hp_peer_reduce) with `world` ranks emulated in one
process on cuda:0: every rank's receive buffers are local, the kernels and
the epoch/flag protocol are the multi-GPU ones.

Bar: bit-identical to the unfused path it replaces -- per rank the swap-AB
GEMM's bf16 partial (HP_EPI_STORE), then an fp32 sum over ranks in rank
order plus the residual, rounded once to bf16 -- and within the bf16
tolerance of an fp32 torch reference."""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_19516_b200.device import lib  # noqa: E402
from paper_2504_19516_b200.device.peer import PeerAllReduce  # noqa: E402

DEV = torch.device("cuda", 0)


def _unfused(xs, ws_t, resid, sms):
    acc = None
    for x, w in zip(xs, ws_t):
        T, K = x.shape
        N = w.shape[0]
        part = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
        nb = lib.gemm_swap_ws_bytes(T, N, K, sms)
        wsb = torch.empty(nb // 4 + 1, dtype=torch.float32, device=DEV)
        cnt = torch.zeros(N // 128 * 8, dtype=torch.int32, device=DEV)
        lib.gemm_swap(x, w, part, wsb, cnt, lib.EPI_STORE, max_ctas=sms)
        acc = part.float() if acc is None else acc + part.float()
    if resid is not None:
        acc = acc + resid.float()
    return acc.to(torch.bfloat16)


def _receive(ranks, outs, epoch, resid):
    """Every rank's receive side, in an order one stream can run: two-shot
    needs every owner's reduce-scatter before any rank's all-gather."""
    if ranks[0].two_shot:
        for r, pr in enumerate(ranks):
            pr.reduce_scatter(outs[r].shape[0], epoch, resid=resid)
        for r, pr in enumerate(ranks):
            pr.all_gather(outs[r], epoch)
    else:
        for r, pr in enumerate(ranks):
            pr.reduce(outs[r], epoch, resid=resid)


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("T", [1, 32, 100, 256])
@pytest.mark.parametrize("sms", [8, 148])
@pytest.mark.parametrize("two_shot", [False, True], ids=["one_shot", "two_shot"])
def test_fused_allreduce_matches_unfused(world, T, sms, two_shot):
    N, K = 1024, 512
    g = torch.Generator(device="cpu").manual_seed(world * 1000 + T + sms)
    ranks = PeerAllReduce.local_group(world, 256, N, DEV, two_shot=two_shot)
    for call in range(3):  # both buffer halves, epochs 1..3
        xs = [torch.randn(T, K, generator=g).to(torch.bfloat16).to(DEV) for _ in range(world)]
        wd = [(torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16) for _ in range(world)]
        ws_t = [lib.tile_weight(w.to(DEV)) for w in wd]
        resid = torch.randn(T, N, generator=g).to(torch.bfloat16).to(DEV) if call != 1 else None
        outs = [torch.full((T, N), float("nan"), dtype=torch.bfloat16, device=DEV) for _ in range(world)]
        epoch = call + 1
        for r in range(world):  # every rank's GEMM, then every rank's receive side (one stream)
            ranks[r].gemm(xs[r], ws_t[r], epoch, max_ctas=sms)
        _receive(ranks, outs, epoch, resid)
        torch.cuda.synchronize()
        ref = _unfused(xs, ws_t, resid, sms)
        for r in range(world):
            assert torch.equal(outs[r], ref), (r, call)
        f32 = sum(x.float() @ w.to(DEV).float().T for x, w in zip(xs, wd))
        if resid is not None:
            f32 = f32 + resid.float()
        assert (outs[0].float() - f32).abs().max().item() <= 0.02 * world ** 0.5 + 0.01 * f32.abs().max().item()


def test_fused_allreduce_linear_epochs_advance():
    """PeerAllReduce.linear on a 1-rank group: epochs advance per call and the
    result equals the unfused bf16 partial + residual."""
    N, K, T = 512, 256, 16
    (pr,) = PeerAllReduce.local_group(1, 64, N, DEV)
    g = torch.Generator(device="cpu").manual_seed(3)
    w = lib.tile_weight((torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16).to(DEV))
    for i in range(5):
        x = torch.randn(T, K, generator=g).to(torch.bfloat16).to(DEV)
        r = torch.randn(T, N, generator=g).to(torch.bfloat16).to(DEV)
        out = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
        pr.linear(x, w, out, resid=r, max_ctas=32)
        torch.cuda.synchronize()
        assert pr.epoch == i + 1
        assert torch.equal(out, _unfused([x], [w], r, 32))


def test_fused_allreduce_rejects_bad_shapes():
    with pytest.raises(ValueError):
        PeerAllReduce.local_group(2, 512, 1024, DEV)
    with pytest.raises(ValueError):
        PeerAllReduce.local_group(9, 16, 1024, DEV)
    (pr,) = PeerAllReduce.local_group(1, 16, 1024, DEV)
    x = torch.zeros(32, 256, dtype=torch.bfloat16, device=DEV)
    w = lib.tile_weight(torch.zeros(1024, 256, dtype=torch.bfloat16, device=DEV))
    with pytest.raises(ValueError):
        pr.gemm(x, w, 1)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("two_shot", [False, True], ids=["one_shot", "two_shot"])
def test_fused_allreduce_device_epochs_replay_in_a_cuda_graph(world, two_shot):
    """device_epoch=True: the epoch lives on the device, so one captured graph
    of every rank's GEMM + reduce replays call after call (alternating buffer
    halves) and stays bit-identical to the unfused path."""
    N, K, T = 1024, 512, 48
    g = torch.Generator(device="cpu").manual_seed(77 + world)
    ranks = PeerAllReduce.local_group(world, 64, N, DEV, device_epoch=True, two_shot=two_shot)
    ws_t = [lib.tile_weight((torch.randn(N, K, generator=g) * 0.05).to(torch.bfloat16).to(DEV))
            for _ in range(world)]
    xs = [torch.empty(T, K, dtype=torch.bfloat16, device=DEV) for _ in range(world)]
    resid = torch.empty(T, N, dtype=torch.bfloat16, device=DEV)
    outs = [torch.empty(T, N, dtype=torch.bfloat16, device=DEV) for _ in range(world)]

    def step():
        for r in range(world):
            ranks[r].gemm(xs[r], ws_t[r], 0, max_ctas=32)
        _receive(ranks, outs, 0, resid)

    def fill():
        for x in xs:
            x.copy_(torch.randn(T, K, generator=g).to(torch.bfloat16))
        resid.copy_(torch.randn(T, N, generator=g).to(torch.bfloat16))

    fill()
    step()  # eager call 1 (also sizes the workspaces before capture)
    torch.cuda.synchronize()
    assert all(torch.equal(o, _unfused(xs, ws_t, resid, 32)) for o in outs)
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(graph, stream=s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    for call in range(4):  # replays = epochs 2..5 (both halves, twice)
        fill()
        graph.replay()
        torch.cuda.synchronize()
        ref = _unfused(xs, ws_t, resid, 32)
        for r in range(world):
            assert torch.equal(outs[r], ref), (call, r)
    for pr in ranks:
        assert pr.epoch_dev[0].item() == 5 and pr.epoch_dev[1].item() == 0
