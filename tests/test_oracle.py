"""Self-checks of the CPU numerics oracle (oracle/numerics.py) against
independent torch-CPU formulations, so the checker itself is trustworthy.

The reference has no transformer numerics (parity unpinned); these
tests pin the oracle to the standard definitions instead.
"""

import math

import numpy as np
import pytest
import torch

from oracle import numerics as O


def test_bf16_round_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([(rng.normal(size=10000) * 10.0 ** rng.integers(-5, 5, 10000)).astype(np.float32),
                        np.array([0.0, -0.0, 1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -9, 65504.0, 3e38], np.float32)])
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(O.bf16_round(x), ref)


def torch_attention(q, k, v, scale, causal):
    Hq, Hkv = q.shape[1], k.shape[1]
    qt = torch.from_numpy(q).permute(1, 0, 2)
    kt = torch.from_numpy(k).repeat_interleave(Hq // Hkv, dim=1).permute(1, 0, 2)
    vt = torch.from_numpy(v).repeat_interleave(Hq // Hkv, dim=1).permute(1, 0, 2)
    s = qt @ kt.transpose(1, 2) * scale
    if causal:
        Tq, Tk = q.shape[0], k.shape[0]
        m = torch.ones(Tq, Tk, dtype=torch.bool).tril(Tk - Tq)
        s = s.masked_fill(~m, float("-inf"))
    return (s.softmax(-1) @ vt).permute(1, 0, 2).numpy()


@pytest.mark.parametrize("T,Hq,Hkv,d,prior", [(37, 4, 2, 64, 0), (80, 8, 1, 128, 0), (20, 4, 4, 64, 30)])
def test_causal_attention_vs_torch(T, Hq, Hkv, d, prior):
    rng = np.random.default_rng(T)
    q = rng.normal(size=(T, Hq, d)).astype(np.float32)
    k = rng.normal(size=(prior + T, Hkv, d)).astype(np.float32)
    v = rng.normal(size=(prior + T, Hkv, d)).astype(np.float32)
    got = O.causal_attention(q, k, v, 1 / math.sqrt(d), prior=prior)
    ref = torch_attention(q, k, v, 1 / math.sqrt(d), True)
    assert np.max(np.abs(got - ref)) < 1e-4


def test_paged_decode_equals_last_row_of_causal():
    rng = np.random.default_rng(1)
    Hq, Hkv, d, page = 8, 2, 64, 64
    ctx = np.array([1, 63, 64, 65, 200])
    B = len(ctx)
    pages = -(-ctx // page)
    nblk = int(pages.sum()) + 2
    kc = rng.normal(size=(nblk, Hkv, page, d)).astype(np.float32)
    vc = rng.normal(size=(nblk, Hkv, page, d)).astype(np.float32)
    perm = rng.permutation(nblk)
    bt = np.zeros((B, pages.max()), dtype=np.int64)
    i = 0
    for b, p in enumerate(pages):
        bt[b, :p] = perm[i:i + p]
        i += p
    q = rng.normal(size=(B, Hq, d)).astype(np.float32)
    got = O.paged_decode_attention(q, kc, vc, bt, ctx, 0.125)
    for b, c in enumerate(ctx):
        k = kc[bt[b, :pages[b]]].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:c]
        v = vc[bt[b, :pages[b]]].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:c]
        ref = torch_attention(q[b:b + 1], k, v, 0.125, False)[0]
        assert np.max(np.abs(got[b] - ref)) < 1e-4


def test_rope_properties():
    d = 128
    table = O.rope_table(5000, d)
    rng = np.random.default_rng(2)
    x = rng.normal(size=(6, 3, d)).astype(np.float32)
    assert np.allclose(O.apply_rope(x, np.zeros(6, int), table), x)
    pos = rng.integers(0, 4000, 6)
    y = O.apply_rope(x, pos, table)
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-5)
    # relative: <R(p)q, R(p+k)k> independent of p
    q, k = x[:1, :1], x[1:2, :1]
    a = (O.apply_rope(q, np.array([10]), table) * O.apply_rope(k, np.array([17]), table)).sum()
    b = (O.apply_rope(q, np.array([1000]), table) * O.apply_rope(k, np.array([1007]), table)).sum()
    assert abs(a - b) < 1e-3


def torch_layer(x, W, Hq, Hkv, d, table):
    """Independent torch restatement of a Llama layer (fp32, no bf16 rounding)."""
    t = lambda a: torch.from_numpy(np.asarray(a, np.float32))  # noqa: E731
    xt = t(x)

    def rms(z, w):
        return z * torch.rsqrt(z.pow(2).mean(-1, keepdim=True) + 1e-5) * t(w)

    T = x.shape[0]
    qkv = rms(xt, W.attn_norm) @ t(W.w_qkv).T
    q = qkv[:, :Hq * d].view(T, Hq, d)
    k = qkv[:, Hq * d:(Hq + Hkv) * d].view(T, Hkv, d)
    v = qkv[:, (Hq + Hkv) * d:].view(T, Hkv, d)
    cos, sin = t(table[:T, :d // 2])[:, None], t(table[:T, d // 2:])[:, None]

    def rot(z):
        z1, z2 = z[..., :d // 2], z[..., d // 2:]
        return torch.cat([z1 * cos - z2 * sin, z2 * cos + z1 * sin], -1)

    q, k = rot(q), rot(k)
    kk = k.repeat_interleave(Hq // Hkv, 1).transpose(0, 1)
    vv = v.repeat_interleave(Hq // Hkv, 1).transpose(0, 1)
    a = torch.nn.functional.scaled_dot_product_attention(q.transpose(0, 1), kk, vv, is_causal=True)
    h = xt + a.transpose(0, 1).reshape(T, Hq * d) @ t(W.w_o).T
    n2 = rms(h, W.mlp_norm)
    act = torch.nn.functional.silu(n2 @ t(W.w_gate).T) * (n2 @ t(W.w_up).T)
    return (h + act @ t(W.w_down).T).numpy()


def test_layer_prefill_vs_torch_restatement():
    rng = np.random.default_rng(3)
    h, Hq, Hkv, d, I, T = 256, 4, 2, 64, 768, 50
    W = O.LayerWeights(rng.normal(0, .02, ((Hq + 2 * Hkv) * d, h)), rng.normal(0, .02, (h, h)),
                       rng.normal(0, .02, (I, h)), rng.normal(0, .02, (I, h)), rng.normal(0, .02, (h, I)),
                       1 + .1 * rng.normal(size=h), 1 + .1 * rng.normal(size=h))
    W = O.LayerWeights(*[np.asarray(a, np.float32) for a in
                         (W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, W.attn_norm, W.mlp_norm)])
    x = rng.normal(size=(T, h)).astype(np.float32)
    table = O.rope_table(T, d)
    y, _, _ = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(T), table, bf16_boundaries=False)
    assert np.max(np.abs(y - torch_layer(x, W, Hq, Hkv, d, table))) < 1e-4


def test_decode_step_consistent_with_prefill():
    """Decoding token t with the cache of tokens < t reproduces prefill row t."""
    rng = np.random.default_rng(4)
    h, Hq, Hkv, d, I, T, page = 256, 4, 2, 64, 768, 70, 64
    W = O.LayerWeights(*[np.asarray(a, np.float32) for a in (
        rng.normal(0, .02, ((Hq + 2 * Hkv) * d, h)), rng.normal(0, .02, (h, h)), rng.normal(0, .02, (I, h)),
        rng.normal(0, .02, (I, h)), rng.normal(0, .02, (h, I)), 1 + .1 * rng.normal(size=h),
        1 + .1 * rng.normal(size=h))])
    x = rng.normal(size=(T, h)).astype(np.float32)
    table = O.rope_table(T + 1, d)
    y, k, v = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(T), table, bf16_boundaries=False)
    kc = np.zeros((2, Hkv, page, d), np.float32)
    vc = np.zeros_like(kc)
    for j in range(T - 1):
        kc[j // page, :, j % page] = k[j]
        vc[j // page, :, j % page] = v[j]
    yd = O.layer_decode(x[T - 1:], W, Hq, Hkv, d, np.array([T]), table, kc, vc, np.array([[0, 1]]),
                        bf16_boundaries=False)
    assert np.max(np.abs(yd[0] - y[T - 1])) < 1e-4


def _tiny_layer(rng, h=64, Hq=4, Hkv=2, d=16, inter=96):
    def w(*s):
        return O.bf16_round((rng.normal(size=s) * 0.05).astype(np.float32))

    return O.LayerWeights(w((Hq + 2 * Hkv) * d, h), w(h, h), w(inter, h), w(inter, h), w(h, inter),
                          O.bf16_round(1 + 0.1 * rng.normal(size=h).astype(np.float32)),
                          O.bf16_round(1 + 0.1 * rng.normal(size=h).astype(np.float32))), Hq, Hkv, d


def test_layer_hybrid_chunked_equals_unchunked_prefill_and_decode():
    # hybrid_kernels (workload.py:213-257): splitting a prompt into chunks with
    # cached prefixes, and packing decode rows beside them, changes nothing
    rng = np.random.default_rng(7)
    W, Hq, Hkv, d = _tiny_layer(rng)
    page, T = 8, 45
    table = O.rope_table(128, d)
    x = O.bf16_round(rng.normal(size=(T, 64)).astype(np.float32))
    ref, _, _ = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(T), table, bf16_boundaries=False)
    nblk = 20
    bt = rng.permutation(nblk)[None, :8]
    kc = np.zeros((nblk, Hkv, page, d), np.float32)
    vc = np.zeros_like(kc)
    parts = []
    for p, n in [(0, 13), (13, 20), (33, 12)]:
        parts.append(O.layer_hybrid(x[p:p + n], W, Hq, Hkv, d, [(n, p)], table, kc, vc, bt,
                                    bf16_boundaries=False))
    np.testing.assert_allclose(np.concatenate(parts), ref, atol=2e-5, rtol=1e-4)
    # a decode row (1, ctx-1) beside a chunk equals layer_decode on the same cache
    xd = O.bf16_round(rng.normal(size=(1, 64)).astype(np.float32))
    kc2, vc2 = kc.copy(), vc.copy()
    bt2 = np.stack([bt[0], rng.permutation(np.arange(8, 20))[:8]])
    xc = O.bf16_round(rng.normal(size=(5, 64)).astype(np.float32))
    hyb = O.layer_hybrid(np.concatenate([xc, xd]), W, Hq, Hkv, d, [(5, 0), (1, T)], table, kc, vc,
                         bt2[::-1].copy(), bf16_boundaries=False)
    dec = O.layer_decode(xd, W, Hq, Hkv, d, np.array([T + 1]), table, kc2, vc2, bt2[:1],
                         bf16_boundaries=False)
    np.testing.assert_allclose(hyb[5:], dec, atol=2e-5, rtol=1e-4)
