"""CPU numerics oracle for the B200 hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module, and only as the checker (or the timed CPU baseline); the
product path (paper_2504_19516_b200) never calls it and has no CPU fallback.

Numerics are not pinnable to the reference: smshare is an analytical
simulator with no transformer arithmetic at all (SPEC.md:18 lists "actual
transformer inference and numerics" as out of scope; pkg/tests holds no
numerics fixtures).  They are pinned instead to an independent
implementation of the same layer -- Hugging Face transformers 5.5's
LlamaDecoderLayer in fp32 (tests/test_oracle_hf.py: prefill layers and a
paged decode step agree to 2e-4 relative).  This restatement follows the reference's
kernel decomposition -- the five groups of `layer_kernels`
(pkg/src/smshare/workload.py:162-210):

  qkv        RMSNorm(x) . W_qkv^T                     (workload.py:164-170)
  attn       causal GQA attention over prefix + span   (workload.py:176-183)
             / paged decode attention over the context (workload.py:184-188)
  o_proj     attn . W_o^T + residual                   (workload.py:191-194)
  mlp_up_gate silu(RMSNorm(h) . W_g^T) * (. W_u^T)     (workload.py:196-204)
  mlp_down   . W_down^T + residual                     (workload.py:205-209)

with the standard Llama definitions for the rest (RMSNorm eps 1e-5,
rotate-half RoPE with theta 500000, SwiGLU), as listed in PAPER.md:6-8.

Arithmetic is numpy float32 with float64 softmax/normalisation sums.  With
``bf16_boundaries=True`` every kernel output is rounded to bfloat16 exactly
where the device stores bf16 (qkv, rope'd q/k, attention output, residual
stream, SwiGLU activations), so the remaining differences are accumulation
order and exp/rsqrt ulps only.
"""

from __future__ import annotations

import math

import numpy as np

EPS = 1e-5
ROPE_THETA = 500000.0


# ------------------------------------------------------------------ bf16
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    a = np.ascontiguousarray(x, dtype=np.float32)
    u = a.view(np.uint32)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    nan = np.isnan(a)
    out = r.view(np.float32).copy()
    out[nan] = np.nan
    return out


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _b(x, on):
    return bf16_round(x) if on else x


# ------------------------------------------------------------------ pieces
def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float = EPS) -> np.ndarray:
    x64 = x.astype(np.float64)
    inv = 1.0 / np.sqrt((x64 * x64).mean(axis=-1, keepdims=True) + eps)
    return (x * inv.astype(np.float32)) * w


def rope_table(max_pos: int, head_dim: int, theta: float = ROPE_THETA) -> np.ndarray:
    """[max_pos, head_dim] float32: cos for the first half, sin for the second
    (computed in float64; the device reads the same table)."""
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def apply_rope(x: np.ndarray, pos: np.ndarray, table: np.ndarray) -> np.ndarray:
    """x [T, H, d]; rotate-half convention."""
    d = x.shape[-1]
    half = d // 2
    cos = table[pos, :half][:, None, :]
    sin = table[pos, half:][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def _softmax_rows(s: np.ndarray) -> np.ndarray:
    s64 = s.astype(np.float64)
    m = s64.max(axis=-1, keepdims=True)
    e = np.exp(s64 - m)
    return (e / e.sum(axis=-1, keepdims=True)).astype(np.float32)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float,
                     prior: int = 0) -> np.ndarray:
    """q [T, Hq, d]; k, v [prior + T, Hkv, d]; query i attends keys <= prior + i."""
    T, Hq, d = q.shape
    Hkv = k.shape[1]
    G = Hq // Hkv
    L = k.shape[0]
    out = np.empty((T, Hq, d), dtype=np.float32)
    mask = np.arange(L)[None, :] <= (prior + np.arange(T))[:, None]
    for h in range(Hq):
        kh, vh = k[:, h // G, :], v[:, h // G, :]
        s = (q[:, h, :] @ kh.T) * scale
        s = np.where(mask, s, -np.inf)
        out[:, h, :] = _softmax_rows(s) @ vh
    return out


def paged_decode_attention(q: np.ndarray, kcache: np.ndarray, vcache: np.ndarray,
                           block_table: np.ndarray, ctx_lens: np.ndarray, scale: float) -> np.ndarray:
    """q [B, Hq, d]; caches [blocks, Hkv, page, d]; one query per sequence over
    its ctx_lens[b] cached positions."""
    B, Hq, d = q.shape
    Hkv, page = kcache.shape[1], kcache.shape[2]
    G = Hq // Hkv
    out = np.empty((B, Hq, d), dtype=np.float32)
    for b in range(B):
        c = int(ctx_lens[b])
        pages = block_table[b, : -(-c // page)]
        k = kcache[pages].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:c]
        v = vcache[pages].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:c]
        for h in range(Hq):
            s = (k[:, h // G, :] @ q[b, h, :]) * scale
            out[b, h, :] = _softmax_rows(s[None, :])[0] @ v[:, h // G, :]
    return out


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x.astype(np.float64))).astype(np.float32)


# ------------------------------------------------------------------ layer
class LayerWeights:
    """One decoder layer's weights as float32 arrays holding bf16 values.

    w_qkv [(Hq+2Hkv) d, h], w_o [h, h], w_gate / w_up [I, h], w_down [h, I],
    attn_norm / mlp_norm [h]."""

    def __init__(self, w_qkv, w_o, w_gate, w_up, w_down, attn_norm, mlp_norm):
        self.w_qkv, self.w_o = w_qkv, w_o
        self.w_gate, self.w_up, self.w_down = w_gate, w_up, w_down
        self.attn_norm, self.mlp_norm = attn_norm, mlp_norm


def layer_prefill(x: np.ndarray, W: LayerWeights, Hq: int, Hkv: int, d: int, pos: np.ndarray,
                  table: np.ndarray, bf16_boundaries: bool = True, trace: dict | None = None):
    """One prefill layer over a single sequence's new span (no cached prefix).

    Returns (y, k_rot, v): the layer output and the K/V rows written to cache.
    `trace`: if a dict, receives the stored intermediates q (roped), attn,
    h (residual after o_proj) and act (SwiGLU output) for per-tensor parity."""
    rb = bf16_boundaries
    T = x.shape[0]
    qkv = _b(_b(rmsnorm(x, W.attn_norm), rb) @ W.w_qkv.T, rb)
    q = qkv[:, : Hq * d].reshape(T, Hq, d)
    k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(T, Hkv, d)
    v = qkv[:, (Hq + Hkv) * d:].reshape(T, Hkv, d)
    q = _b(apply_rope(q, pos, table), rb)
    k = _b(apply_rope(k, pos, table), rb)
    a = _b(causal_attention(q, k, v, 1.0 / math.sqrt(d)).reshape(T, Hq * d), rb)
    h = _b(x + a @ W.w_o.T, rb)
    n2 = _b(rmsnorm(h, W.mlp_norm), rb)
    act = _b(silu(n2 @ W.w_gate.T) * (n2 @ W.w_up.T), rb)
    y = _b(h + act @ W.w_down.T, rb)
    if trace is not None:
        trace.update(q=q.reshape(T, Hq * d), attn=a, h=h, act=act)
    return y, k, v


def layer_decode(x: np.ndarray, W: LayerWeights, Hq: int, Hkv: int, d: int, ctx_lens: np.ndarray,
                 table: np.ndarray, kcache: np.ndarray, vcache: np.ndarray, block_table: np.ndarray,
                 bf16_boundaries: bool = True, trace: dict | None = None) -> np.ndarray:
    """One decode layer step for B sequences: the new token of sequence b sits
    at position ctx_lens[b]-1; its K/V are written into the (mutated) caches
    before attention over ctx_lens[b] positions.  `trace`: as layer_prefill."""
    rb = bf16_boundaries
    B = x.shape[0]
    page = kcache.shape[2]
    pos = (np.asarray(ctx_lens) - 1).astype(np.int64)
    qkv = _b(_b(rmsnorm(x, W.attn_norm), rb) @ W.w_qkv.T, rb)
    q = _b(apply_rope(qkv[:, : Hq * d].reshape(B, Hq, d), pos, table), rb)
    k = _b(apply_rope(qkv[:, Hq * d:(Hq + Hkv) * d].reshape(B, Hkv, d), pos, table), rb)
    v = qkv[:, (Hq + Hkv) * d:].reshape(B, Hkv, d)
    for b in range(B):
        blk = block_table[b, pos[b] // page]
        kcache[blk, :, pos[b] % page, :] = k[b]
        vcache[blk, :, pos[b] % page, :] = v[b]
    a = _b(paged_decode_attention(q, kcache, vcache, block_table, ctx_lens,
                                  1.0 / math.sqrt(d)).reshape(B, Hq * d), rb)
    h = _b(x + a @ W.w_o.T, rb)
    n2 = _b(rmsnorm(h, W.mlp_norm), rb)
    act = _b(silu(n2 @ W.w_gate.T) * (n2 @ W.w_up.T), rb)
    if trace is not None:
        trace.update(q=q.reshape(B, Hq * d), attn=a, h=h, act=act)
    return _b(h + act @ W.w_down.T, rb)


def layer_hybrid(x: np.ndarray, W: LayerWeights, Hq: int, Hkv: int, d: int, seqs, table: np.ndarray,
                 kcache: np.ndarray, vcache: np.ndarray, block_table: np.ndarray,
                 bf16_boundaries: bool = True) -> np.ndarray:
    """One layer over a hybrid (chunked-prefill) batch -- reference
    hybrid_kernels (workload.py:213-257): linear kernels over the
    concatenated token stream, attention per sequence over its cached prefix
    plus its new span (workload.py:176-183).

    seqs[i] = (new_len, prior) in row order of x; sequence i's pages are
    block_table[i].  A decode token is (1, ctx - 1).  The new tokens' K/V are
    written into the (mutated) caches before attention."""
    rb = bf16_boundaries
    T = x.shape[0]
    page = kcache.shape[2]
    pos = np.concatenate([np.arange(p, p + n) for n, p in seqs]).astype(np.int64)
    assert len(pos) == T
    qkv = _b(_b(rmsnorm(x, W.attn_norm), rb) @ W.w_qkv.T, rb)
    q = _b(apply_rope(qkv[:, : Hq * d].reshape(T, Hq, d), pos, table), rb)
    k = _b(apply_rope(qkv[:, Hq * d:(Hq + Hkv) * d].reshape(T, Hkv, d), pos, table), rb)
    v = qkv[:, (Hq + Hkv) * d:].reshape(T, Hkv, d)
    a = np.empty((T, Hq, d), np.float32)
    r0 = 0
    for i, (n, p) in enumerate(seqs):
        for j in range(n):
            blk = block_table[i, (p + j) // page]
            kcache[blk, :, (p + j) % page, :] = k[r0 + j]
            vcache[blk, :, (p + j) % page, :] = v[r0 + j]
        L = p + n
        pages = block_table[i, : -(-L // page)]
        kk = kcache[pages].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:L]
        vv = vcache[pages].transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:L]
        a[r0:r0 + n] = causal_attention(q[r0:r0 + n], kk, vv, 1.0 / math.sqrt(d), prior=p)
        r0 += n
    a = _b(a.reshape(T, Hq * d), rb)
    h = _b(x + a @ W.w_o.T, rb)
    n2 = _b(rmsnorm(h, W.mlp_norm), rb)
    act = _b(silu(n2 @ W.w_gate.T) * (n2 @ W.w_up.T), rb)
    return _b(h + act @ W.w_down.T, rb)


def greedy_tokens(hidden: np.ndarray, final_norm: np.ndarray, lm_head: np.ndarray,
                  bf16_boundaries: bool = True):
    """argmax over logits = RMSNorm(hidden) . lm_head^T; also the top-2 margin."""
    n = _b(rmsnorm(hidden, final_norm), bf16_boundaries)
    logits = _b(n @ lm_head.T, bf16_boundaries)  # the device stores logits as bf16
    top2 = np.sort(logits, axis=-1)[:, -2:]
    return logits.argmax(axis=-1), top2[:, 1] - top2[:, 0], logits
