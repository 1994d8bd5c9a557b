"""Tensor-parallel decoder layer (BASELINE config 5: Llama-3-70B, TP = 8,
chunked prefill 2048 + decode batch 128).

Megatron split of one layer over `world` GPUs, one process per GPU:

  qkv          column-parallel: rank r owns q heads [r Hq/w, (r+1) Hq/w) and
               kv heads [r Hkv/w, ...) -> attention is head-local, no exchange
  o_proj       row-parallel over the attention output columns; partial sums
               (rank 0 folds in the residual) -> all-reduce #1
  mlp_up_gate  column-parallel over the intermediate dim (gate/up of the same
               rows stay together, 64-row interleave as in the 1-GPU layer)
  mlp_down     row-parallel; partials (+ residual on rank 0) -> all-reduce #2

so a layer costs two all-reduces of T x hidden bf16 (32 MiB at T = 2048,
hidden 8192).  The all-reduces run on the calling stream through the given
process group (NCCL over NVLink / NVSwitch on a B200 node), i.e. on the same
green-context partition as the phase's kernels, which is where the
reference charges collective traffic (the n_w term, perf_model.py:172-180).
All compute is the 1-GPU hot path's kernels on the local shapes.

With `peer=` (a PeerAllReduce, device/peer.py) decode-sized steps
(T <= peer.T_max) skip both collectives: o_proj and mlp_down scatter their
partial tiles into every rank's receive buffer from the GEMM epilogue and a
flag-gated reduce adds the residual.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import lib
from .layer import EPS, interleave_gate_up, rope_table

PAGE = 64


@dataclass(frozen=True)
class TPShape:
    hidden: int
    heads: int      # local q heads
    kv_heads: int   # local kv heads
    head_dim: int
    inter: int      # local intermediate

    @property
    def qkv_out(self) -> int:
        return (self.heads + 2 * self.kv_heads) * self.head_dim


def tp_shape(hidden: int, Hq: int, Hkv: int, d: int, inter: int, world: int) -> TPShape:
    if Hq % world or Hkv % world or inter % world:
        raise ValueError(f"heads {Hq}/{Hkv} and intermediate {inter} must divide by world {world}")
    return TPShape(hidden, Hq // world, Hkv // world, d, inter // world)


def shard_dense(w_qkv, w_o, w_gate, w_up, w_down, Hq: int, Hkv: int, d: int, rank: int, world: int):
    """Rank `rank`'s slices of [out, in] weights (numpy or torch): returns
    (w_qkv_l, w_o_l, w_gate_l, w_up_l, w_down_l)."""
    hq, hk = Hq // world, Hkv // world
    q = w_qkv[rank * hq * d:(rank + 1) * hq * d]
    k = w_qkv[Hq * d + rank * hk * d: Hq * d + (rank + 1) * hk * d]
    v = w_qkv[(Hq + Hkv) * d + rank * hk * d:(Hq + Hkv) * d + (rank + 1) * hk * d]
    cat = torch.cat if isinstance(w_qkv, torch.Tensor) else __import__("numpy").concatenate
    inter = w_gate.shape[0] // world
    return (cat([q, k, v]), w_o[:, rank * hq * d:(rank + 1) * hq * d], w_gate[rank * inter:(rank + 1) * inter],
            w_up[rank * inter:(rank + 1) * inter], w_down[:, rank * inter:(rank + 1) * inter])


class TPLayer:
    """One layer's shard resident on this rank's GPU plus its launch sequences."""

    def __init__(self, shape: TPShape, w_qkv_l, w_o_l, w_gate_l, w_up_l, w_down_l, attn_norm, mlp_norm,
                 rank: int, group=None, device=None, max_tokens: int = 4096, max_pos: int = 32768,
                 allreduce=None, peer=None):
        """`allreduce(tensor)` overrides the collective (default:
        torch.distributed.all_reduce over `group` on the calling stream)."""
        self.s = shape
        self.allreduce = allreduce
        self.peer = peer
        self.rank = rank
        self.group = group
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        t = lib.tile_weight
        self.w_qkv, self.w_o = t(w_qkv_l), t(w_o_l)
        self.w_ug, self.w_down = t(interleave_gate_up(w_gate_l, w_up_l)), t(w_down_l)
        self.attn_norm, self.mlp_norm = attn_norm, mlp_norm
        self.scale = 1.0 / math.sqrt(shape.head_dim)
        self.rope = torch.from_numpy(rope_table(max_pos, shape.head_dim)).to(self.dev)
        bf = dict(dtype=torch.bfloat16, device=self.dev)
        h = shape.hidden
        self.xn = torch.empty(max_tokens, h, **bf)
        self.qkv = torch.empty(max_tokens, shape.qkv_out, **bf)
        self.attn = torch.empty(max_tokens, shape.heads * shape.head_dim, **bf)
        self.h = torch.empty(max_tokens, h, **bf)
        self.act = torch.empty(max_tokens, shape.inter, **bf)
        self.max_tokens = max_tokens
        self._sw = None

    def _allreduce(self, t, stream):
        st = torch.cuda.ExternalStream(stream) if isinstance(stream, int) else stream
        with torch.cuda.stream(st or torch.cuda.current_stream()):
            if self.allreduce is not None:
                self.allreduce(t)
            elif self.group is not None:
                import torch.distributed as dist

                dist.all_reduce(t, group=self.group)

    def _epi(self):
        # residual folded in once (rank 0) so the all-reduce sum holds it once
        return lib.EPI_RESID if self.rank == 0 else lib.EPI_STORE

    def _swap_ws(self, T):
        if self._sw is None:
            s = self.s
            shapes = [(s.qkv_out, s.hidden), (s.hidden, s.heads * s.head_dim), (2 * s.inter, s.hidden),
                      (s.hidden, s.inter)]
            nb = max(lib.gemm_swap_ws_bytes(256, n, k, c) for n, k in shapes for c in (1, 148))
            self._sw = (torch.empty(nb // 4 + 1, dtype=torch.float32, device=self.dev),
                        torch.zeros(max(n for n, _ in shapes) // 128 * 8, dtype=torch.int32, device=self.dev))
        return self._sw

    def _linear(self, x, w, y, epi, resid, sms, stream):
        if x.shape[0] <= 256:
            ws, cnt = self._swap_ws(x.shape[0])
            lib.gemm_swap(x, w, y, ws, cnt, epi, resid=resid, max_ctas=sms, stream=stream)
        else:
            lib.gemm(x, w, y, epi, resid=resid, max_ctas=sms, stream=stream)

    def prefill(self, x, y, cu_seqlens, nseq, max_seqlen, positions, slots, kcache, vcache, sms, stream=None):
        """y = layer(x) for packed new tokens x [T, hidden] (replicated on every
        rank); K/V of the local kv heads go to this rank's cache shard."""
        s, T = self.s, x.shape[0]
        d = s.head_dim
        lib.rmsnorm(x, self.attn_norm, self.xn[:T], EPS, sms, stream)
        q = self.qkv[:T]
        if T > 256:  # fused GEMM + RoPE + paged K/V write
            lib.gemm_qkv_rope(self.xn[:T], self.w_qkv, q, s.heads, s.kv_heads, d, positions, self.rope, slots,
                              kcache, vcache, PAGE, max_ctas=sms, stream=stream)
        else:
            self._linear(self.xn[:T], self.w_qkv, q, lib.EPI_STORE, None, sms, stream)
            lib.rope_kv_write(q, s.heads, s.kv_heads, d, positions, self.rope, slots, kcache, vcache, PAGE,
                              max_ctas=sms, stream=stream)
        lib.prefill_attn(q[:, :s.heads * d], q[:, s.heads * d:(s.heads + s.kv_heads) * d],
                         q[:, (s.heads + s.kv_heads) * d:], self.attn[:T], cu_seqlens, nseq, max_seqlen,
                         s.heads, s.kv_heads, d, self.scale, max_ctas=sms, stream=stream)
        return self._tail(x, y, T, sms, stream)

    def decode(self, x, y, ctx_lens, positions, slots, block_table, kcache, vcache, sms, stream=None, ws=None):
        s, B = self.s, x.shape[0]
        d = s.head_dim
        lib.rmsnorm(x, self.attn_norm, self.xn[:B], EPS, sms, stream)
        self._linear(self.xn[:B], self.w_qkv, self.qkv[:B], lib.EPI_STORE, None, sms, stream)
        lib.rope_kv_write(self.qkv[:B], s.heads, s.kv_heads, d, positions, self.rope, slots, kcache, vcache,
                          PAGE, max_ctas=sms, stream=stream)
        lib.decode_attn(self.qkv[:B], kcache, vcache, block_table, ctx_lens, self.attn[:B], s.heads, s.kv_heads,
                        d, PAGE, self.scale, ws=ws, max_ctas=sms, stream=stream)
        return self._tail(x, y, B, sms, stream)

    def _tail(self, x, y, T, sms, stream):
        if self.peer is not None and T <= self.peer.T_max:
            # fused: every rank adds the (replicated) residual in the reduce
            self.peer.linear(self.attn[:T], self.w_o, self.h[:T], resid=x, max_ctas=sms, stream=stream)
            lib.rmsnorm(self.h[:T], self.mlp_norm, self.xn[:T], EPS, sms, stream)
            self._linear(self.xn[:T], self.w_ug, self.act[:T], lib.EPI_SILU, None, sms, stream)
            self.peer.linear(self.act[:T], self.w_down, y, resid=self.h[:T], max_ctas=sms, stream=stream)
            return 0
        epi = self._epi()
        self._linear(self.attn[:T], self.w_o, self.h[:T], epi, x if epi == lib.EPI_RESID else None, sms, stream)
        self._allreduce(self.h[:T], stream)                    # all-reduce #1 (post O-proj)
        lib.rmsnorm(self.h[:T], self.mlp_norm, self.xn[:T], EPS, sms, stream)
        self._linear(self.xn[:T], self.w_ug, self.act[:T], lib.EPI_SILU, None, sms, stream)
        self._linear(self.act[:T], self.w_down, y, epi, self.h[:T] if epi == lib.EPI_RESID else None, sms, stream)
        self._allreduce(y, stream)                             # all-reduce #2 (post down-proj)
        return 2
