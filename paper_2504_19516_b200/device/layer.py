"""One Llama decoder layer on the B200: weights, KV cache, and the prefill /
decode launch sequences over libb200hot.so.

The five device launches per pass are the five kernel groups of the
reference's layer API (`layer_kernels`, workload.py:162-210), in order:

  qkv          rmsnorm + tcgen05 GEMM (prefill: RoPE + paged-KV write fused
               into the GEMM epilogue, token-major prefill and swap-AB decode alike)
  attn         causal GQA flash attention (prefill) | paged decode attention
  o_proj       tcgen05 GEMM with fused residual add
  mlp_up_gate  rmsnorm + tcgen05 GEMM with fused SiLU(gate) * up
  mlp_down     tcgen05 GEMM with fused residual add

Prefill uses the token-major GEMM (grid = output tiles, persistent over the
partition's SMs); decode uses the swap-AB stream-K GEMM.  Every launch takes
the partition's SM count as its grid size, so a launch issued into a
green-context stream of `pm` SMs is exactly the "layer on pm SMs" the
reference's oracle call stands for (engine.py:189-198).

Data layout in HBM (bf16 unless noted):
  x / h / y          [T, hidden] residual stream (ping-pong, inputs untouched)
  qkv                [T, (Hq + 2 Hkv) d]  q | k | v column blocks
  w_qkv              [(Hq + 2 Hkv) d, hidden]        torch [out, in], then tiled
  w_o                [hidden, hidden]                 (hp_tile_weight: [N/128][K/128][2]
  w_ug               [2 I, hidden]  gate/up rows       128B-swizzled,
                     interleaved in 64-row blocks      [128][64], so each 128x128 tile is one
  w_down             [hidden, I]                       contiguous bulk copy)
  kcache / vcache    [num_blocks, Hkv, page, d] logical; stored per page as
                     [page/64][d/64][64][64] (64-token tiles, each one
                     contiguous run) with swizzled 16B chunks (lib.kv_pack);
                     zero-initialised
  block_table int32  [B, max_pages];  ctx_lens int32 [B]
  rope table fp32    [max_pos, d]  (cos | sin)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ..workload import ModelSpec
from . import lib

PAGE = 64
EPS = 1e-5


def mlp_width(model: ModelSpec) -> int:
    """MLP rows materialised on the device.  The reference approximates a
    sparse MoE by scaling the MLP's weights, FLOPs and intermediate
    activations by `activated_fraction` (workload.py:26-38, 76-79, 196-209);
    the device realises that as a dense SwiGLU MLP of width
    intermediate x activated_fraction, rounded to the 128-row weight tile
    (moe-a22b: 1228.8 -> 1280).  Dense presets: exactly `intermediate`."""
    f = model.activated_fraction
    if f == 1.0:
        return model.intermediate
    return max(128, int(round(model.intermediate * f / 128)) * 128)
ROPE_THETA = 500000.0


def rope_table(max_pos: int, head_dim: int, theta: float = ROPE_THETA) -> np.ndarray:
    """float64-computed cos|sin table, stored fp32 (same table the CPU oracle uses)."""
    inv = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor, block: int = 64) -> torch.Tensor:
    """[I, h] x 2 -> [2I, h] with rows [g0..g63, u0..u63, g64.., ...]."""
    inter, h = w_gate.shape
    assert inter % block == 0
    return torch.stack([w_gate.view(-1, block, h), w_up.view(-1, block, h)], dim=1).reshape(2 * inter, h)


@dataclass
class LayerWeights:
    w_qkv: torch.Tensor
    w_o: torch.Tensor
    w_ug: torch.Tensor
    w_down: torch.Tensor
    attn_norm: torch.Tensor
    mlp_norm: torch.Tensor

    @classmethod
    def random(cls, model: ModelSpec, device, gen: torch.Generator, std: float = 0.02):
        h, I = model.hidden, mlp_width(model)

        def w(*shape):
            return (torch.randn(*shape, generator=gen, device="cpu") * std).to(torch.bfloat16).to(device)

        def norm():
            return (1.0 + 0.1 * torch.randn(h, generator=gen, device="cpu")).to(torch.bfloat16).to(device)

        gate, up = w(I, h), w(I, h)
        return cls.from_dense(w(model.qkv_out_dim, h), w(h, h), gate, up, w(h, I), norm(), norm())

    @classmethod
    def random_device(cls, model: ModelSpec, device, gen: torch.Generator, std: float = 0.02):
        """Random weights drawn on the GPU (a 32-layer model's 14 GB would take
        minutes through the host generator)."""
        h, I = model.hidden, mlp_width(model)

        def w(*shape):
            return (torch.randn(*shape, generator=gen, device=device) * std).to(torch.bfloat16)

        def norm():
            return (1.0 + 0.1 * torch.randn(h, generator=gen, device=device)).to(torch.bfloat16)

        return cls.from_dense(w(model.qkv_out_dim, h), w(h, h), w(I, h), w(I, h), w(h, I), norm(), norm())

    @classmethod
    def from_dense(cls, w_qkv, w_o, w_gate, w_up, w_down, attn_norm, mlp_norm):
        """Row-major torch [out, in] device weights -> the resident layout:
        gate/up interleaved, every matrix tiled for bulk-copy streaming."""
        t = lib.tile_weight
        out = cls(t(w_qkv), t(w_o), t(interleave_gate_up(w_gate, w_up)), t(w_down), attn_norm, mlp_norm)
        torch.cuda.synchronize()
        return out

    @classmethod
    def from_numpy(cls, device, w_qkv, w_o, w_gate, w_up, w_down, attn_norm, mlp_norm):
        def t(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(device)

        return cls.from_dense(t(w_qkv), t(w_o), t(w_gate), t(w_up), t(w_down), t(attn_norm), t(mlp_norm))

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.w_qkv, self.w_o, self.w_ug, self.w_down, self.attn_norm, self.mlp_norm))


class KVCache:
    """Paged K/V for one layer: [num_blocks, Hkv, page, d] bf16 each."""

    def __init__(self, num_blocks: int, Hkv: int, d: int, device, page: int = PAGE):
        self.page = page
        self.k = torch.zeros(num_blocks, Hkv, page, d, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros_like(self.k)

    @property
    def num_blocks(self) -> int:
        return self.k.shape[0]


class PrefillScratch:
    """Activation buffers for a prefill pass of up to `max_tokens` tokens."""

    def __init__(self, model: ModelSpec, max_tokens: int, device):
        h = model.hidden
        bf = dict(dtype=torch.bfloat16, device=device)
        self.max_tokens = max_tokens
        self.xn = torch.empty(max_tokens, h, **bf)
        self.qkv = torch.empty(max_tokens, model.qkv_out_dim, **bf)
        self.attn = torch.empty(max_tokens, h, **bf)
        self.h = torch.empty(max_tokens, h, **bf)
        self.act = torch.empty(max_tokens, mlp_width(model), **bf)


class DecodeScratch:
    """Activation buffers + stream-K workspaces for a decode batch of <= max_batch."""

    def __init__(self, model: ModelSpec, max_batch: int, max_pages: int, device, max_ctas: int = 148):
        h, I = model.hidden, mlp_width(model)
        bf = dict(dtype=torch.bfloat16, device=device)
        self.max_batch = max_batch
        self.xn = torch.empty(max_batch, h, **bf)
        self.qkv = torch.empty(max_batch, model.qkv_out_dim, **bf)
        self.attn = torch.empty(max_batch, h, **bf)
        self.h = torch.empty(max_batch, h, **bf)
        self.act = torch.empty(max_batch, I, **bf)
        shapes = [(model.qkv_out_dim, h), (h, h), (2 * I, h), (h, I)]
        ws = max(lib.gemm_swap_ws_bytes(max_batch, n, k, c) for n, k in shapes
                 for c in range(1, max(max_ctas, 148) + 1))
        self.gemm_ws = torch.empty(ws // 4 + 1, dtype=torch.float32, device=device)
        n_cnt = max(n // 128 for n, _ in shapes) * 8
        self.gemm_cnt = torch.zeros(n_cnt, dtype=torch.int32, device=device)
        splits = 4 * max_pages + 8
        self.attn_ws = torch.empty(lib.decode_attn_ws_bytes(max_batch, model.num_heads, model.head_dim,
                                                            splits) // 4 + 1,
                                   dtype=torch.float32, device=device)


class DeviceLayer:
    """A Llama layer resident in HBM plus its launch sequences."""

    def __init__(self, model: ModelSpec, weights: LayerWeights, device, max_pos: int = 32768):
        self.model = model
        self.W = weights
        self.device = device
        self.Hq, self.Hkv, self.d = model.num_heads, model.num_kv_heads, model.head_dim
        self.scale = 1.0 / math.sqrt(self.d)
        self.rope = torch.from_numpy(rope_table(max_pos, self.d)).to(device)

    # -------------------------------------------------------------- prefill
    def prefill(self, x, y, sc: PrefillScratch, cu_seqlens, nseq: int, max_seqlen: int,
                positions, slots, cache: KVCache, sms: int, stream=None, timers=None, cta_trace=None) -> int:
        """y = layer(x) for the packed prefill tokens of x [T, h]; writes the
        sequences' K/V into `cache` at `slots`.  Returns the launch count.
        `timers`: optional {kernel group: (start_event, end_event)} recorded on
        `stream` around that group's main launch (qkv, attn, o_proj,
        mlp_up_gate, mlp_down).  `cta_trace`: optional {group: int64 [grid, 3]}
        receiving that launch's per-CTA {smid, start_ns, end_ns}."""
        T = x.shape[0]
        qkv = sc.qkv[:T]
        Hq, Hkv, d = self.Hq, self.Hkv, self.d
        timers = timers or {}
        rs = stream if stream is not None else torch.cuda.current_stream().cuda_stream

        cta_trace = cta_trace or {}

        def mark(name, i):
            ev = timers.get(name)
            if ev is not None:
                ev[i].record(torch.cuda.ExternalStream(rs) if isinstance(rs, int) else rs)
            if i == 0 and name in cta_trace:
                lib.arm_cta_trace(cta_trace[name])

        lib.rmsnorm(x, self.W.attn_norm, sc.xn[:T], EPS, sms, stream)
        mark("qkv", 0)
        # QKV GEMM with RoPE + the paged K/V write fused into its epilogue
        lib.gemm_qkv_rope(sc.xn[:T], self.W.w_qkv, qkv, Hq, Hkv, d, positions, self.rope, slots, cache.k,
                          cache.v, cache.page, max_ctas=sms, stream=stream)
        mark("qkv", 1)
        mark("attn", 0)
        lib.prefill_attn(qkv[:, : Hq * d], qkv[:, Hq * d:(Hq + Hkv) * d], qkv[:, (Hq + Hkv) * d:],
                         sc.attn[:T], cu_seqlens, nseq, max_seqlen, Hq, Hkv, d, self.scale,
                         max_ctas=sms, stream=stream)
        mark("attn", 1)
        mark("o_proj", 0)
        lib.gemm(sc.attn[:T], self.W.w_o, sc.h[:T], lib.EPI_RESID, resid=x, max_ctas=sms, stream=stream)
        mark("o_proj", 1)
        lib.rmsnorm(sc.h[:T], self.W.mlp_norm, sc.xn[:T], EPS, sms, stream)
        mark("mlp_up_gate", 0)
        lib.gemm(sc.xn[:T], self.W.w_ug, sc.act[:T], lib.EPI_SILU, max_ctas=sms, stream=stream)
        mark("mlp_up_gate", 1)
        mark("mlp_down", 0)
        lib.gemm(sc.act[:T], self.W.w_down, y, lib.EPI_RESID, resid=sc.h[:T], max_ctas=sms, stream=stream)
        mark("mlp_down", 1)
        return 7

    # --------------------------------------------------------------- decode
    def decode(self, x, y, sc: DecodeScratch, ctx_lens, positions, slots, block_table,
               cache: KVCache, sms: int, stream=None) -> int:
        """One decode step of this layer for B = x.shape[0] sequences; the new
        token of sequence b is at positions[b] (= ctx_lens[b] - 1), its K/V go
        to slots[b].  Returns the launch count (decode attention may add a
        split-combine launch)."""
        B = x.shape[0]
        m = self.model
        Hq, Hkv, d = self.Hq, self.Hkv, self.d
        ws, cnt = sc.gemm_ws, sc.gemm_cnt
        qkv = sc.qkv[:B]
        lib.rmsnorm(x, self.W.attn_norm, sc.xn[:B], EPS, sms, stream)
        lib.gemm_swap_qkv_rope(sc.xn[:B], self.W.w_qkv, qkv, Hq, Hkv, d, positions, self.rope, slots, cache.k,
                               cache.v, cache.page, ws, cnt, max_ctas=sms, stream=stream)
        lib.decode_attn(qkv, cache.k, cache.v, block_table, ctx_lens, sc.attn[:B], Hq, Hkv, d,
                        cache.page, self.scale, ws=sc.attn_ws, max_ctas=sms, stream=stream)
        lib.gemm_swap(sc.attn[:B], self.W.w_o, sc.h[:B], ws, cnt, lib.EPI_RESID, resid=x,
                      max_ctas=sms, stream=stream)
        lib.rmsnorm(sc.h[:B], self.W.mlp_norm, sc.xn[:B], EPS, sms, stream)
        lib.gemm_swap(sc.xn[:B], self.W.w_ug, sc.act[:B], ws, cnt, lib.EPI_SILU, max_ctas=sms,
                      stream=stream)
        lib.gemm_swap(sc.act[:B], self.W.w_down, y, ws, cnt, lib.EPI_RESID, resid=sc.h[:B],
                      max_ctas=sms, stream=stream)
        return 7 + lib.decode_attn_launches(B, Hq, Hkv, d, block_table.shape[1], cache.page, sms)


    # --------------------------------------------------------------- hybrid
    def hybrid(self, x, y, sc: PrefillScratch, dsc: DecodeScratch, n_chunk_tokens: int, cu_chunks,
               n_chunks: int, max_chunk: int, prior_lens, chunk_block_table, dec_ctx_lens, dec_block_table,
               positions, slots, cache: KVCache, sms: int, stream=None) -> int:
        """One layer over a hybrid batch (the lockstep chunked-prefill
        baseline; reference hybrid_kernels workload.py:213-257): rows
        [0, n_chunk_tokens) of x are prefill-chunk tokens of `n_chunks`
        sequences (offsets cu_chunks, cached prefixes prior_lens, pages
        chunk_block_table), the remaining B rows are decode tokens (contexts
        dec_ctx_lens incl. the new token, pages dec_block_table).  The four
        linear kernels run once over the concatenated stream; attention is
        prefix-aware paged prefill attention for the chunks plus paged decode
        attention for the decode rows.  positions/slots cover all rows.
        Returns the launch count."""
        T = x.shape[0]
        Tc = n_chunk_tokens
        B = T - Tc
        if T > sc.max_tokens or B > dsc.max_batch or Tc < 0:
            raise ValueError(f"hybrid batch of {Tc} chunk + {B} decode rows exceeds the scratch "
                             f"({sc.max_tokens} rows, {dsc.max_batch} decode)")
        Hq, Hkv, d = self.Hq, self.Hkv, self.d
        qkv = sc.qkv[:T]
        swap = T <= dsc.max_batch

        def linear(inp, w, out, epi, resid=None):
            if swap:
                lib.gemm_swap(inp, w, out, dsc.gemm_ws, dsc.gemm_cnt, epi, resid=resid, max_ctas=sms,
                              stream=stream)
            else:
                lib.gemm(inp, w, out, epi, resid=resid, max_ctas=sms, stream=stream)

        n = 0
        lib.rmsnorm(x, self.W.attn_norm, sc.xn[:T], EPS, sms, stream)
        if swap:  # RoPE + paged K/V write fused into the swap GEMM's epilogue
            lib.gemm_swap_qkv_rope(sc.xn[:T], self.W.w_qkv, qkv, Hq, Hkv, d, positions, self.rope, slots,
                                   cache.k, cache.v, cache.page, dsc.gemm_ws, dsc.gemm_cnt, max_ctas=sms,
                                   stream=stream)
            n += 2
        else:  # token-major GEMM with RoPE + paged K/V write fused into the epilogue
            lib.gemm_qkv_rope(sc.xn[:T], self.W.w_qkv, qkv, Hq, Hkv, d, positions, self.rope, slots, cache.k,
                              cache.v, cache.page, max_ctas=sms, stream=stream)
            n += 2
        if Tc > 0:
            lib.prefill_attn_paged(qkv[:Tc, : Hq * d], cache.k, cache.v, chunk_block_table, cu_chunks,
                                   prior_lens, n_chunks, max_chunk, sc.attn[:Tc], Hq, Hkv, d, cache.page,
                                   self.scale, max_ctas=sms, stream=stream)
            n += 1
        if B > 0:
            lib.decode_attn(qkv[Tc:], cache.k, cache.v, dec_block_table, dec_ctx_lens, sc.attn[Tc:T], Hq,
                            Hkv, d, cache.page, self.scale, ws=dsc.attn_ws, max_ctas=sms, stream=stream)
            n += 1
        linear(sc.attn[:T], self.W.w_o, sc.h[:T], lib.EPI_RESID, resid=x)
        lib.rmsnorm(sc.h[:T], self.W.mlp_norm, sc.xn[:T], EPS, sms, stream)
        linear(sc.xn[:T], self.W.w_ug, sc.act[:T], lib.EPI_SILU)
        linear(sc.act[:T], self.W.w_down, y, lib.EPI_RESID, resid=sc.h[:T])
        return n + 4


def decode_slots(block_table: torch.Tensor, ctx_lens: torch.Tensor, page: int = PAGE):
    """positions = ctx-1 and cache slots of each sequence's newest token."""
    pos = (ctx_lens - 1).to(torch.int64)
    blk = torch.gather(block_table.to(torch.int64), 1, (pos // page)[:, None])[:, 0]
    return pos.to(torch.int32), (blk * page + pos % page).to(torch.int32)
