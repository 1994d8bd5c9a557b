"""Kernel-level numerics of libb200hot.so against torch fp32 references.

Floating-point kernels are compared with a plain fp32 restatement of the same
op (bf16 inputs upcast); tolerances are stated per test.  Run on a B200 with
`pytest -m gpu`.
"""

import math

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2504_19516_b200.device import lib  # noqa: E402

DEV = torch.device("cuda", 0)


def rel_err(got, ref):
    got = got.float()
    ref = ref.float()
    return ((got - ref).abs().max() / ref.abs().max().clamp_min(1e-6)).item()


def bf(shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen, device=DEV) * scale).to(torch.bfloat16)


@pytest.fixture(scope="module")
def gen():
    g = torch.Generator(device=DEV)
    g.manual_seed(1234)
    return g


# ------------------------------------------------------------------- GEMM
@pytest.mark.parametrize("T,N,K", [(128, 256, 256), (200, 768, 512), (1024, 6144, 4096),
                                   (77, 4096, 4096), (4096, 1024, 1024)])
def test_gemm_store(T, N, K, gen):
    x, w = bf((T, K), gen=gen), bf((N, K), 0.05, gen)
    y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    lib.gemm(x, lib.tile_weight(w),y, lib.EPI_STORE, max_ctas=148)
    ref = x.float() @ w.float().T
    torch.cuda.synchronize()
    assert rel_err(y, ref) < 1e-2


def test_prefill_gemm_and_attention_bitwise_invariant_to_partition_and_batch(gen):
    # the co-run and the time-sliced baseline must compute the same numbers:
    # prefill GEMM outputs (no split-K below 128 k-blocks) and prefill
    # attention outputs do not depend on the SM partition, nor -- for the
    # GEMM -- on which other rows share the call
    T, N, K = 1024, 4096, 4096
    x, w = bf((T, K), gen=gen), bf((N, K), 0.05, gen)
    wt = lib.tile_weight(w)
    outs = []
    for sms in (148, 140, 52, 16):
        y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
        lib.gemm(x, wt, y, lib.EPI_STORE, max_ctas=sms)
        outs.append(y)
    for y in outs[1:]:
        assert torch.equal(outs[0], y)
    y256 = torch.empty(256, N, device=DEV, dtype=torch.bfloat16)
    lib.gemm(x[256:512].contiguous(), wt, y256, lib.EPI_STORE, max_ctas=148)
    assert torch.equal(outs[0][256:512], y256)
    Hq, Hkv, d = 32, 8, 128
    qkv = bf((T, (Hq + 2 * Hkv) * d), gen=gen)
    q, kk, vv = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    cu = torch.tensor([0, T], dtype=torch.int32, device=DEV)
    att = []
    for sms in (148, 124, 8):
        o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
        lib.prefill_attn(q, kk, vv, o, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=sms)
        att.append(o)
    for o in att[1:]:
        assert torch.equal(att[0], o)


@pytest.mark.parametrize("max_ctas", [1, 16, 148])
def test_gemm_grid_sizes(max_ctas, gen):
    T, N, K = 300, 512, 640
    x, w = bf((T, K), gen=gen), bf((N, K), 0.05, gen)
    y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    lib.gemm(x, lib.tile_weight(w),y, lib.EPI_STORE, max_ctas=max_ctas)
    assert rel_err(y, x.float() @ w.float().T) < 1e-2


def test_gemm_resid(gen):
    T, N, K = 333, 4096, 1024
    x, w, r = bf((T, K), gen=gen), bf((N, K), 0.05, gen), bf((T, N), gen=gen)
    y = torch.empty_like(r)
    lib.gemm(x, lib.tile_weight(w),y, lib.EPI_RESID, resid=r)
    assert rel_err(y, x.float() @ w.float().T + r.float()) < 1e-2
    # in place (out aliases the residual), as the layer uses it
    r2 = r.clone()
    lib.gemm(x, lib.tile_weight(w),r2, lib.EPI_RESID, resid=r2)
    assert rel_err(r2, x.float() @ w.float().T + r.float()) < 1e-2


def silu_ref(z):
    return z * torch.sigmoid(z)


def interleave_ref(N2, K, gen):
    """Weight with gate/up rows interleaved in blocks of 64, plus the plain halves."""
    g, u = bf((N2, K), 0.05, gen), bf((N2, K), 0.05, gen)
    w = torch.stack([g.view(-1, 64, K), u.view(-1, 64, K)], dim=1).reshape(2 * N2, K)
    return w.contiguous(), g, u


@pytest.mark.parametrize("T", [64, 257])
def test_gemm_silu(T, gen):
    N2, K = 1024, 512
    w, g, u = interleave_ref(N2, K, gen)
    x = bf((T, K), gen=gen)
    y = torch.empty(T, N2, device=DEV, dtype=torch.bfloat16)
    lib.gemm(x, lib.tile_weight(w),y, lib.EPI_SILU)
    ref = silu_ref(x.float() @ g.float().T) * (x.float() @ u.float().T)
    assert rel_err(y, ref) < 2e-2


def _ws(N, T, K, ctas):
    bn = 32 if T <= 32 else 64 if T <= 64 else 128 if T <= 128 else 256
    ws = torch.empty(lib.gemm_swap_ws_bytes(T, N, K, ctas) // 4, device=DEV, dtype=torch.float32)
    cnt = torch.zeros((N // 128) * (-(-T // bn)), device=DEV, dtype=torch.int32)
    return ws, cnt


@pytest.mark.parametrize("T,N,K,ctas", [(1, 256, 256, 1), (8, 6144, 4096, 148), (32, 4096, 4096, 64),
                                        (32, 4096, 4096, 32), (33, 1024, 1024, 7), (100, 512, 2048, 148),
                                        (256, 256, 512, 3), (32, 28672, 4096, 148),
                                        # CTA-pair kernel (N % 256 == 0 on <= 16 SMs): BN 32 / 64 / 128 /
                                        # 256, split and whole tiles, tokens past T zero-filled
                                        (32, 4096, 4096, 8), (20, 6144, 4096, 16), (64, 512, 2048, 2),
                                        (100, 1024, 1024, 6), (256, 512, 512, 4), (9, 28672, 4096, 8)])
def test_gemm_swap_store(T, N, K, ctas, gen):
    x, w = bf((T, K), gen=gen), bf((N, K), 0.05, gen)
    y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    ws, cnt = _ws(N, T, K, ctas)
    lib.gemm_swap(x, lib.tile_weight(w),y, ws, cnt, lib.EPI_STORE, max_ctas=ctas)
    assert rel_err(y, x.float() @ w.float().T) < 1e-2
    # arrival counters are left clean for the next call
    torch.cuda.synchronize()
    assert cnt.abs().max().item() == 0
    y.zero_()
    lib.gemm_swap(x, lib.tile_weight(w),y, ws, cnt, lib.EPI_STORE, max_ctas=ctas)
    assert rel_err(y, x.float() @ w.float().T) < 1e-2


@pytest.mark.parametrize("ctas", [32, 148, 8, 2])
def test_gemm_swap_resid_silu(ctas, gen):
    T, K = 32, 1024
    x, r = bf((T, K), gen=gen), bf((T, 4096), gen=gen)
    w = bf((4096, K), 0.05, gen)
    ws, cnt = _ws(4096, T, K, ctas)
    y = r.clone()
    lib.gemm_swap(x, lib.tile_weight(w),y, ws, cnt, lib.EPI_RESID, resid=y, max_ctas=ctas)
    assert rel_err(y, x.float() @ w.float().T + r.float()) < 1e-2
    wi, g, u = interleave_ref(1024, K, gen)
    ws2, cnt2 = _ws(2048, T, K, ctas)
    y2 = torch.empty(T, 1024, device=DEV, dtype=torch.bfloat16)
    lib.gemm_swap(x, lib.tile_weight(wi), y2, ws2, cnt2, lib.EPI_SILU, max_ctas=ctas)
    ref = silu_ref(x.float() @ g.float().T) * (x.float() @ u.float().T)
    assert rel_err(y2, ref) < 2e-2


@pytest.mark.parametrize("ctas", [8, 148])
def test_gemm_swap_row_independent_within_a_batch_bucket(ctas, gen):
    # serving determinism: a decode request's output rows must not depend on
    # which other requests share its step -- within one token bucket (same
    # BN, hence the same stream-K split and fp32 summation order) the first
    # 13 rows of a 32-row call equal a 13-row call bit for bit
    N, K = 4096, 4096
    x, w = bf((32, K), gen=gen), bf((N, K), 0.05, gen)
    wt = lib.tile_weight(w)
    ws, cnt = _ws(N, 32, K, ctas)
    y32 = torch.empty(32, N, device=DEV, dtype=torch.bfloat16)
    y13 = torch.empty(13, N, device=DEV, dtype=torch.bfloat16)
    lib.gemm_swap(x, wt, y32, ws, cnt, lib.EPI_STORE, max_ctas=ctas)
    lib.gemm_swap(x[:13].contiguous(), wt, y13, ws, cnt, lib.EPI_STORE, max_ctas=ctas)
    assert torch.equal(y32[:13], y13)


# ------------------------------------------------------------- RMSNorm / RoPE
def test_rmsnorm(gen):
    x, wt = bf((77, 4096), gen=gen), bf((4096,), 1.0, gen)
    out = torch.empty_like(x)
    lib.rmsnorm(x, wt, out, 1e-5, max_ctas=16)
    xf = x.float()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * wt.float()
    assert rel_err(out, ref) < 1e-2


def rope_table(max_pos, d, theta=500000.0):
    inv = 1.0 / (theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
    ang = torch.arange(max_pos, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cat([ang.cos(), ang.sin()], dim=1).float().to(DEV)


@pytest.mark.parametrize("page", [64, 128])
def test_rope_kv_write(gen, page):
    T, Hq, Hkv, d = 100, 8, 2, 128
    qkv = bf((T, (Hq + 2 * Hkv) * d), gen=gen)
    orig = qkv.float().clone()
    pos = torch.randint(0, 4000, (T,), device=DEV, dtype=torch.int32)
    nblk = 8
    slots = torch.randperm(nblk * page, device=DEV)[:T].to(torch.int32)
    kc = torch.zeros(nblk, Hkv, page, d, device=DEV, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    cs = rope_table(4096, d)
    lib.rope_kv_write(qkv, Hq, Hkv, d, pos, cs, slots, kc, vc, page)
    cos, sin = cs[pos.long(), : d // 2], cs[pos.long(), d // 2:]

    def rot(x):  # [T, H, d]
        x1, x2 = x[..., : d // 2], x[..., d // 2:]
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)

    o3 = orig.view(T, Hq + 2 * Hkv, d)
    q_ref, k_ref, v_ref = rot(o3[:, :Hq]), rot(o3[:, Hq:Hq + Hkv]), o3[:, Hq + Hkv:]
    got = qkv.float().view(T, Hq + 2 * Hkv, d)
    assert rel_err(got[:, :Hq], q_ref) < 1e-2
    assert rel_err(got[:, Hq:Hq + Hkv], k_ref) < 1e-2
    blk, off = (slots // page).long(), (slots % page).long()
    kc, vc = lib.kv_unpack(kc), lib.kv_unpack(vc)  # device page layout -> logical
    assert rel_err(kc[blk, :, off], k_ref) < 1e-2
    assert torch.equal(vc[blk, :, off].float(), v_ref)


# ------------------------------------------------------------- attention
def attn_ref(q, k, v, causal, scale):
    """q [Tq, Hq, d], k/v [Tk, Hkv, d] fp32; causal aligns the last query to the last key."""
    Hq, Hkv = q.shape[1], k.shape[1]
    k = k.repeat_interleave(Hq // Hkv, dim=1)
    v = v.repeat_interleave(Hq // Hkv, dim=1)
    s = torch.einsum("qhd,khd->hqk", q, k) * scale
    if causal:
        Tq, Tk = q.shape[0], k.shape[0]
        mask = torch.ones(Tq, Tk, dtype=torch.bool, device=q.device).tril(Tk - Tq)
        s = s.masked_fill(~mask, float("-inf"))
    return torch.einsum("hqk,khd->qhd", s.softmax(-1), v)


@pytest.mark.parametrize("lens,Hq,Hkv,d", [([128], 4, 1, 128), ([1000], 8, 2, 128),
                                           ([64, 130, 7], 4, 4, 128), ([2048], 32, 8, 128),
                                           ([1024], 4, 2, 64), ([5, 300], 4, 2, 64), ([700], 64, 4, 64)])
def test_prefill_attn(lens, Hq, Hkv, d, gen):
    T = sum(lens)
    qkv = bf((T, (Hq + 2 * Hkv) * d), gen=gen)
    q, k, v = qkv[:, : Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    o = torch.zeros(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), device=DEV, dtype=torch.int32)
    scale = 1.0 / math.sqrt(d)
    lib.prefill_attn(q, k, v, o, cu, len(lens), max(lens), Hq, Hkv, d, scale)
    s0 = 0
    for L in lens:
        sl = slice(s0, s0 + L)
        ref = attn_ref(q[sl].float().view(L, Hq, d), k[sl].float().view(L, Hkv, d),
                       v[sl].float().view(L, Hkv, d), True, scale)
        got = o[sl].float().view(L, Hq, d)
        assert (got - ref).abs().max().item() < 2e-2
        s0 += L


def make_cache(B, ctx, Hkv, d, page, gen, extra_blocks=3):
    pages = [-(-c // page) for c in ctx]
    nblk = sum(pages) + extra_blocks
    kc = bf((nblk, Hkv, page, d), gen=gen)
    vc = bf((nblk, Hkv, page, d), gen=gen)
    perm = torch.randperm(nblk, device=DEV).to(torch.int32)
    max_pages = max(pages)
    bt = torch.zeros(B, max_pages, device=DEV, dtype=torch.int32)
    i = 0
    for b, p in enumerate(pages):
        bt[b, :p] = perm[i:i + p]
        i += p
    return kc, vc, bt


@pytest.mark.parametrize("ctx,Hq,Hkv,d", [([17, 64, 128, 255, 256, 511, 512, 1000], 4, 2, 128),
                                          ([2048] * 32, 32, 8, 128), ([1], 8, 1, 128),
                                          ([5000, 33], 64, 8, 128), ([3000] * 3, 32, 8, 128),
                                          ([17, 64, 128, 255, 256, 511, 512, 1000], 4, 2, 64),
                                          # GQA 16 (moe-a22b: 64 q / 4 kv heads, d 64) and 24: head blocks
                                          ([2048] * 4 + [100, 7], 64, 4, 64), ([700, 1], 48, 2, 128),
                                          ([300, 64], 32, 1, 64), ([500], 32, 2, 128)])
@pytest.mark.parametrize("max_ctas", [8, 148])
@pytest.mark.parametrize("page", [64, 256])
def test_decode_attn(ctx, Hq, Hkv, d, max_ctas, page, gen):
    B = len(ctx)
    kc, vc, bt = make_cache(B, ctx, Hkv, d, page, gen)
    q = bf((B, Hq * d), gen=gen)
    out = torch.zeros(B, Hq * d, device=DEV, dtype=torch.bfloat16)
    ctx_t = torch.tensor(ctx, device=DEV, dtype=torch.int32)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 256) // 4, device=DEV, dtype=torch.float32)
    scale = 1.0 / math.sqrt(d)
    lib.decode_attn(q, lib.kv_pack(kc), lib.kv_pack(vc), bt, ctx_t, out, Hq, Hkv, d, page, scale,
                    ws=ws, max_ctas=max_ctas)
    for b, c in enumerate(ctx):
        np_ = -(-c // page)
        blocks = bt[b, :np_].long()
        k = kc[blocks].permute(0, 2, 1, 3).reshape(-1, Hkv, d)[:c].float()
        v = vc[blocks].permute(0, 2, 1, 3).reshape(-1, Hkv, d)[:c].float()
        ref = attn_ref(q[b].float().view(1, Hq, d), k, v, False, scale)
        got = out[b].float().view(1, Hq, d)
        assert (got - ref).abs().max().item() < 2e-2, f"seq {b} ctx {c}"


@pytest.mark.parametrize("max_ctas", [8, 148])
def test_decode_attn_single_token_context_is_exact_v(max_ctas, gen):
    # a sequence whose context is one cached token must return that token's V
    # bit for bit (softmax weight exactly 1; any masked slot of the partial
    # tile leaking in, or a stale ring slot, breaks equality), beside long
    # neighbours that keep the ring and the split path busy
    Hq, Hkv, d, page = 32, 8, 128, 64
    ctx = [1, 2048, 1, 777, 1]
    B = len(ctx)
    kc, vc, bt = make_cache(B, ctx, Hkv, d, page, gen)
    q = bf((B, Hq * d), gen=gen)
    out = torch.zeros(B, Hq * d, device=DEV, dtype=torch.bfloat16)
    ctx_t = torch.tensor(ctx, device=DEV, dtype=torch.int32)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 256) // 4, device=DEV, dtype=torch.float32)
    lib.decode_attn(q, lib.kv_pack(kc), lib.kv_pack(vc), bt, ctx_t, out, Hq, Hkv, d, page,
                    1.0 / math.sqrt(d), ws=ws, max_ctas=max_ctas)
    for b, c in enumerate(ctx):
        if c != 1:
            continue
        v0 = vc[bt[b, 0].long(), :, 0, :]  # [Hkv, d]: token 0 of the sequence's first page
        want = v0.repeat_interleave(Hq // Hkv, 0).reshape(-1)
        assert torch.equal(out[b], want), b


def test_decode_attn_page_placement_invariant(gen):
    # the same logical K/V placed on different physical pages (another block
    # table) must give bit-identical outputs
    Hq, Hkv, d, page = 32, 8, 128, 64
    ctx = [2048, 700, 1, 64, 129]
    B = len(ctx)
    kc, vc, bt = make_cache(B, ctx, Hkv, d, page, gen)
    q = bf((B, Hq * d), gen=gen)
    ctx_t = torch.tensor(ctx, device=DEV, dtype=torch.int32)
    ws = torch.empty(lib.decode_attn_ws_bytes(B, Hq, d, 256) // 4, device=DEV, dtype=torch.float32)
    out1 = torch.zeros(B, Hq * d, device=DEV, dtype=torch.bfloat16)
    lib.decode_attn(q, lib.kv_pack(kc), lib.kv_pack(vc), bt, ctx_t, out1, Hq, Hkv, d, page, 1 / math.sqrt(d),
                    ws=ws, max_ctas=148)
    # move every block to a new physical slot
    nblk = kc.shape[0]
    perm = torch.randperm(nblk, device=DEV)
    kc2, vc2 = torch.empty_like(kc), torch.empty_like(vc)
    kc2[perm], vc2[perm] = kc, vc
    bt2 = perm.to(torch.int32)[bt.long()]
    out2 = torch.zeros_like(out1)
    lib.decode_attn(q, lib.kv_pack(kc2), lib.kv_pack(vc2), bt2, ctx_t, out2, Hq, Hkv, d, page, 1 / math.sqrt(d),
                    ws=ws, max_ctas=148)
    assert torch.equal(out1, out2)


# ------------------------------------------------------------- partitions
def test_wave_stats_native():
    assert lib.wave_stats(216, 2, 108) == (1, 108, 0.0)
    assert lib.wave_stats(110, 1, 108) == (2, 2, 106 / 216)
    assert lib.wave_stats(384, 1, 148) == (3, 88, (148 - 88) / (148 * 3))


def test_partition_confinement():
    n = lib.device_sms(0)
    part = lib.Partition(16)
    assert part.decode_sms == 16 and part.prefill_sms == n - 16
    outs = {}
    for phase in (0, 1):
        buf = torch.zeros(4 * n, 3, device=DEV, dtype=torch.int64)
        lib.probe(buf, 4 * n, spin_ns=50000, stream=part.raw_stream(phase))
        torch.cuda.synchronize()
        outs[phase] = set(buf[:, 0].tolist())
    assert len(outs[1]) <= 16
    assert len(outs[0]) <= n - 16
    assert not (outs[0] & outs[1])
    part.close()


def test_partition_confinement_under_graph_replay():
    """Kernels replayed from a CUDA graph captured on a green-context stream
    stay on that partition's SMs (decode steps are graph-replayed)."""
    n = lib.device_sms(0)
    part = lib.Partition(24)
    st = part.stream(1)
    buf = torch.zeros(4 * n, 3, device=DEV, dtype=torch.int64)
    with torch.cuda.stream(st):
        lib.probe(buf, 4 * n, spin_ns=20000, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            lib.probe(buf, 4 * n, spin_ns=20000, stream=st)
        buf.zero_()
        g.replay()
    torch.cuda.synchronize()
    sms = set(buf[:, 0].tolist())
    assert len(sms) <= 24, sorted(sms)
    part.close()


# --------------------------------------------------- paged prefill attention
def _paged_ref(q, kc_logical, vc_logical, bt, lens, priors, scale, G):
    """fp32 reference: sequence s's rows attend cache positions <= prior+i."""
    outs = []
    r0 = 0
    page = kc_logical.shape[2]
    for s, (n, p) in enumerate(zip(lens, priors)):
        L = p + n
        pages = bt[s, : -(-L // page)].long()
        k = kc_logical[pages].permute(0, 2, 1, 3).reshape(-1, kc_logical.shape[1], kc_logical.shape[3])[:L]
        v = vc_logical[pages].permute(0, 2, 1, 3).reshape(-1, vc_logical.shape[1], vc_logical.shape[3])[:L]
        qs = q[r0:r0 + n].float()
        kk = k.float().repeat_interleave(G, dim=1)
        vv = v.float().repeat_interleave(G, dim=1)
        sc = torch.einsum("thd,lhd->htl", qs, kk) * scale
        mask = torch.arange(L, device=DEV)[None, :] <= (p + torch.arange(n, device=DEV))[:, None]
        sc = sc.masked_fill(~mask[None], float("-inf"))
        outs.append(torch.einsum("htl,lhd->thd", sc.softmax(-1), vv))
        r0 += n
    return torch.cat(outs)


@pytest.mark.parametrize("d,Hq,Hkv,lens,priors", [
    (128, 32, 8, [384, 77, 1], [0, 1000, 4095]),
    (128, 32, 8, [1024], [2048]),
    (64, 4, 2, [200, 129, 64], [17, 0, 300]),
    (64, 4, 2, [1], [0]),
])
def test_prefill_attn_paged(d, Hq, Hkv, lens, priors, gen):
    page = 64
    G = Hq // Hkv
    need = [-(-(n + p) // page) for n, p in zip(lens, priors)]
    nblk = sum(need) + 3
    perm = torch.randperm(nblk, generator=torch.Generator().manual_seed(5))
    bt = torch.zeros(len(lens), max(need), dtype=torch.int32)
    k = 0
    for i, nb in enumerate(need):
        bt[i, :nb] = perm[k:k + nb]
        k += nb
    bt = bt.to(DEV)
    kc = bf((nblk, Hkv, page, d), gen=gen)
    vc = bf((nblk, Hkv, page, d), gen=gen)
    T = sum(lens)
    q = bf((T, Hq * d), gen=gen)
    o = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device=DEV)
    pr = torch.tensor(priors, dtype=torch.int32, device=DEV)
    scale = 1 / math.sqrt(d)
    lib.prefill_attn_paged(q, lib.kv_pack(kc), lib.kv_pack(vc), bt, cu, pr, len(lens), max(lens), o, Hq, Hkv,
                           d, page, scale, max_ctas=148)
    ref = _paged_ref(q.view(T, Hq, d), kc, vc, bt, lens, priors, scale, G).reshape(T, Hq * d)
    assert rel_err(o, ref) < 2e-2


def test_prefill_attn_paged_matches_dense_without_prefix(gen):
    # prior_lens = 0: the paged path must agree with the dense (qkv-view) kernel
    from paper_2504_19516_b200.device.layer import KVCache

    T, Hq, Hkv, d, page = 700, 32, 8, 128, 64
    qkv = bf((T, (Hq + 2 * Hkv) * d), gen=gen)
    q, kk, vv = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    cu = torch.tensor([0, T], dtype=torch.int32, device=DEV)
    o_dense = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    lib.prefill_attn(q, kk, vv, o_dense, cu, 1, T, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=148)
    pages = -(-T // page)
    cache = KVCache(pages, Hkv, d, DEV)
    kl = torch.zeros(pages * page, Hkv, d, device=DEV, dtype=torch.bfloat16)
    vl = torch.zeros_like(kl)
    kl[:T] = kk.reshape(T, Hkv, d)
    vl[:T] = vv.reshape(T, Hkv, d)
    cache.k.copy_(lib.kv_pack(kl.view(pages, page, Hkv, d).permute(0, 2, 1, 3).contiguous()))
    cache.v.copy_(lib.kv_pack(vl.view(pages, page, Hkv, d).permute(0, 2, 1, 3).contiguous()))
    bt = torch.arange(pages, dtype=torch.int32, device=DEV)[None]
    o_paged = torch.empty_like(o_dense)
    lib.prefill_attn_paged(q, cache.k, cache.v, bt, cu, torch.zeros(1, dtype=torch.int32, device=DEV), 1, T,
                           o_paged, Hq, Hkv, d, page, 1 / math.sqrt(d), max_ctas=148)
    assert torch.equal(o_paged, o_dense)


@pytest.mark.parametrize("seq_lens", [[700], [130, 257, 64, 1], [8448]])
def test_prefill_attn_first_query_row_is_exact_v(seq_lens, gen):
    # causal query 0 of every sequence sees only key 0: softmax weight exactly
    # 1, so its output must equal V row 0 bit for bit on both operand paths
    # (catches any leak of masked keys or a stale / partially landed V tile)
    from paper_2504_19516_b200.device.layer import KVCache

    Hq, Hkv, d, page = 32, 8, 128, 64
    T = sum(seq_lens)
    qkv = bf((T, (Hq + 2 * Hkv) * d), gen=gen)
    q, kk, vv = qkv[:, :Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:]
    starts = [0]
    for n in seq_lens:
        starts.append(starts[-1] + n)
    cu = torch.tensor(starts, dtype=torch.int32, device=DEV)
    nseq, maxlen = len(seq_lens), max(seq_lens)
    o_dense = torch.empty(T, Hq * d, device=DEV, dtype=torch.bfloat16)
    lib.prefill_attn(q, kk, vv, o_dense, cu, nseq, maxlen, Hq, Hkv, d, 1 / math.sqrt(d), max_ctas=148)
    # paged: each sequence in its own pages, no prefix
    ppages = [-(-n // page) for n in seq_lens]
    cache = KVCache(sum(ppages), Hkv, d, DEV)
    kl = torch.zeros(sum(ppages) * page, Hkv, d, device=DEV, dtype=torch.bfloat16)
    vl = torch.zeros_like(kl)
    bt = torch.zeros(nseq, max(ppages), dtype=torch.int32, device=DEV)
    p0 = 0
    for i, n in enumerate(seq_lens):
        kl[p0 * page:p0 * page + n] = kk[starts[i]:starts[i + 1]].reshape(n, Hkv, d)
        vl[p0 * page:p0 * page + n] = vv[starts[i]:starts[i + 1]].reshape(n, Hkv, d)
        bt[i, :ppages[i]] = torch.arange(p0, p0 + ppages[i], dtype=torch.int32, device=DEV)
        p0 += ppages[i]
    npg = sum(ppages)
    cache.k.copy_(lib.kv_pack(kl.view(npg, page, Hkv, d).permute(0, 2, 1, 3).contiguous()))
    cache.v.copy_(lib.kv_pack(vl.view(npg, page, Hkv, d).permute(0, 2, 1, 3).contiguous()))
    o_paged = torch.empty_like(o_dense)
    lib.prefill_attn_paged(q, cache.k, cache.v, bt, cu, torch.zeros(nseq, dtype=torch.int32, device=DEV), nseq,
                           maxlen, o_paged, Hq, Hkv, d, page, 1 / math.sqrt(d), max_ctas=148)
    for s0 in starts[:-1]:
        v0 = vv[s0].view(Hkv, d).repeat_interleave(Hq // Hkv, 0).reshape(-1)
        assert torch.equal(o_dense[s0], v0)
        assert torch.equal(o_paged[s0], v0)


@pytest.mark.parametrize("T,Hq,Hkv,d", [(300, 32, 8, 128), (1024, 4, 2, 64), (77, 8, 2, 128)])
def test_gemm_qkv_rope_fused_matches_fp32(T, Hq, Hkv, d, gen):
    # hp_gemm_qkv_rope: QKV GEMM + RoPE + paged K/V write in one epilogue
    from paper_2504_19516_b200.device.layer import KVCache, rope_table

    K, page = 512, 64
    N = (Hq + 2 * Hkv) * d
    x, w = bf((T, K), gen=gen), bf((N, K), 0.05, gen)
    pos = torch.randint(0, 4000, (T,), device=DEV, dtype=torch.int32, generator=gen)
    nblk = -(-T // page) + 4
    slots = torch.randperm(nblk * page, device=DEV, generator=gen)[:T].to(torch.int32)
    table = torch.from_numpy(rope_table(4096, d)).to(DEV)
    cache = KVCache(nblk, Hkv, d, DEV)
    y = torch.empty(T, N, device=DEV, dtype=torch.bfloat16)
    lib.gemm_qkv_rope(x, lib.tile_weight(w), y, Hq, Hkv, d, pos, table, slots, cache.k, cache.v, page, max_ctas=148)
    ref = (x.float() @ w.float().T).view(T, Hq + 2 * Hkv, d)
    cs = table[pos.long()]
    cos, sin = cs[:, None, : d // 2], cs[:, None, d // 2:]
    a, b = ref[:, : Hq + Hkv, : d // 2], ref[:, : Hq + Hkv, d // 2:]
    rot = torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)
    ref = torch.cat([rot, ref[:, Hq + Hkv:]], dim=1)
    assert rel_err(y.view(T, -1, d), ref) < 1e-2
    kl, vl = lib.kv_unpack(cache.k).float(), lib.kv_unpack(cache.v).float()
    blk, off = (slots // page).long(), (slots % page).long()
    assert rel_err(kl[blk, :, off], ref[:, Hq:Hq + Hkv]) < 1e-2
    assert rel_err(vl[blk, :, off], ref[:, Hq + Hkv:]) < 1e-2
    assert torch.equal(kl[blk, :, off].to(torch.bfloat16), y.view(T, -1, d)[:, Hq:Hq + Hkv])


def test_gemm_qkv_rope_bit_identical_to_unfused_path(gen):
    from paper_2504_19516_b200.device.layer import KVCache, rope_table

    T, Hq, Hkv, d, K, page = 513, 32, 8, 128, 1024, 64
    N = (Hq + 2 * Hkv) * d
    x, w = bf((T, K), gen=gen), lib.tile_weight(bf((N, K), 0.05, gen))
    pos = torch.arange(T, device=DEV, dtype=torch.int32) + 7
    slots = torch.arange(T, device=DEV, dtype=torch.int32) + 64
    table = torch.from_numpy(rope_table(2048, d)).to(DEV)
    c1, c2 = KVCache(-(-T // page) + 2, Hkv, d, DEV), KVCache(-(-T // page) + 2, Hkv, d, DEV)
    y1, y2 = (torch.empty(T, N, device=DEV, dtype=torch.bfloat16) for _ in range(2))
    lib.gemm_qkv_rope(x, w, y1, Hq, Hkv, d, pos, table, slots, c1.k, c1.v, page, max_ctas=148)
    lib.gemm(x, w, y2, lib.EPI_STORE, max_ctas=148)
    lib.rope_kv_write(y2, Hq, Hkv, d, pos, table, slots, c2.k, c2.v, page, max_ctas=148)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(c1.k, c2.k) and torch.equal(c1.v, c2.v)


# ------------------------------------------------------- zero-copy row copy
@pytest.mark.parametrize("rows,cols,ctas", [(32, 4096, 8), (7, 136, 1), (256, 4096, 148)])
def test_copy_rows_pinned_host_both_ways(rows, cols, ctas, gen):
    """hp_copy_rows reads and writes pinned host memory through UVA (the
    decode step's per-step input / output in the end-to-end co-run)."""
    src = bf((rows, cols), gen=gen)
    host = torch.empty(rows, cols, dtype=torch.bfloat16, pin_memory=True)
    lib.copy_rows(src, host, max_ctas=ctas)           # device -> pinned host
    torch.cuda.synchronize()
    assert torch.equal(host, src.cpu())
    dst = torch.zeros(rows, 2 * cols, dtype=torch.bfloat16, device=DEV)[:, cols // 2: cols // 2 + cols]
    if (cols // 2) % 8 == 0:
        lib.copy_rows(host, dst, max_ctas=ctas)       # pinned host -> strided device view
        torch.cuda.synchronize()
        assert torch.equal(dst, src)
