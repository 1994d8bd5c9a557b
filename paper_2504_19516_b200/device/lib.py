"""ctypes binding of ``libb200hot.so`` (the C ABI declared in include/hp.h).

This module is the only place Python touches the native library.  There is no
fallback: if the library is missing or a call fails, `HotPathError` is raised
with the library's own error string.  Tensor helpers accept torch tensors and
pass raw device pointers plus the current (or given) CUDA stream.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from ..errors import InvalidArgumentError

LIB_PATH = Path(__file__).resolve().parent.parent / "_lib" / "libb200hot.so"

EPI_STORE, EPI_RESID, EPI_SILU, EPI_PEER = 0, 1, 2, 3
MAX_PEERS = 8
IPC_HANDLE_BYTES = 64

# Every symbol include/hp.h declares, with (restype, argtypes).
_i, _u64, _p, _f, _sz, _i64 = C.c_int, C.c_uint64, C.c_void_p, C.c_float, C.c_size_t, C.c_int64
SIGNATURES = {
    "hp_abi_version": (_i, []),
    "hp_last_error": (C.c_char_p, []),
    "hp_device_count": (_i, []),
    "hp_device_sms": (_i, [_i, C.POINTER(_i)]),
    "hp_wave_stats": (_i, [_i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(C.c_double)]),
    "hp_partition_create": (_i, [_i, _i, C.POINTER(_p)]),
    "hp_partition_stream": (_i, [_p, _i, C.POINTER(_p)]),
    "hp_partition_sms": (_i, [_p, _i, C.POINTER(_i)]),
    "hp_partition_destroy": (_i, [_p]),
    "hp_rmsnorm": (_i, [_p, _i, _p, _p, _i, _i, _i, _f, _i, _p]),
    "hp_tile_weight": (_i, [_p, _i, _p, _i, _i, _p]),
    "hp_gemm": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _i, _p]),
    "hp_gemm_traced": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _i, _p, _p]),
    "hp_gemm_tiles": (_i, [_i, _i]),
    "hp_gemm_qkv_rope": (_i, [_p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _i, _i, _p]),
    "hp_gemm_plan": (_i, [_i, _i, _i, _i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "hp_gemm_swap": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _p, _sz, _p, _i, _i, _p]),
    "hp_gemm_swap_qkv_rope": (_i, [_p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _i, _p, _sz, _p,
                                   _i, _i, _p]),
    "hp_gemm_swap_ws_bytes": (_sz, [_i, _i, _i, _i]),
    "hp_peer_tiles": (_i, [_i, _i]),
    "hp_gemm_swap_peer": (_i, [_p, _i, _p, _i, _i, _i, _i, _p, _sz, _p, _sz, _i, _i, _i, _p, _i, _p, _sz, _p, _i,
                               _i, _p]),
    "hp_peer_rs": (_i, [_p, _sz, _p, _sz, _p, _sz, _p, _sz, _i, _i, _i, _i, _i, _p, _p, _i, _p]),
    "hp_peer_ag": (_i, [_p, _sz, _p, _sz, _i, _i, _i, _p, _p, _p, _i, _p]),
    "hp_peer_reduce": (_i, [_p, _sz, _p, _sz, _i, _i, _i, _i, _p, _p, _p, _i, _p, _i, _p]),
    "hp_ipc_handle": (_i, [_p, _p, C.POINTER(_sz)]),
    "hp_ipc_open": (_i, [_p, C.POINTER(_p)]),
    "hp_ipc_close": (_i, [_p]),
    "hp_rope_kv_write": (_i, [_p, _i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _i, _i, _p]),
    "hp_prefill_attn": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _p, _i, _i, _i, _i, _i, _i, _f, _i, _p]),
    "hp_set_trace": (_i, [_i, _p]),
    "hp_set_gemm_tail": (_i, [_i]),
    "hp_gemm_tail_reserve": (_i, [_p]),
    "hp_prefill_attn_paged": (_i, [_p, _i, _p, _p, _p, _i, _p, _p, _i, _i, _i, _p, _i, _i, _i, _i, _i, _i, _f,
                                   _i, _p]),
    "hp_decode_attn_ws_bytes": (_sz, [_i, _i, _i, _i]),
    "hp_decode_attn_launches": (_i, [_i, _i, _i, _i, _i, _i, _i]),
    "hp_decode_attn": (_i, [_p, _i, _p, _p, _p, _i, _p, _p, _i, _i, _i, _i, _i, _i, _i, _f, _p, _sz, _i, _p]),
    "hp_copy_rows": (_i, [_p, C.c_long, _p, C.c_long, _i, _i, _i, _p]),
    "hp_probe": (_i, [_i, _i, _i64, _p, _p]),
    "hp_membw": (_i, [_p, _sz, _i, _i, _p, _p]),
    "hp_membw2d": (_i, [_p, _i, _i, _i, _i, _p, _p]),
    "hp_membw_pipe": (_i, [_p, _sz, _i, _i, _i, _p, _p]),
    "hp_membw_ldg": (_i, [_p, _sz, _i, _i, _i, _i, _p, _p]),
    "hp_membw_pfldg": (_i, [_p, _sz, _i, _i, _i, _i, _p, _p]),
    "hp_membw_stage": (_i, [_p, _sz, _i, _i, _i, _i, _i, _p, _p]),
    "hp_hmma_rate": (_i, [_i, _i, _i, _i, _p, _p]),
    "hp_membw_mix": (_i, [_p, _sz, _i, _i, _i, _p, _p]),
    "hp_umma2_rate": (_i, [_i, _i, _i, _p, _p]),
    "hp_umma_rate": (_i, [_i, _i, _i, _i, _p, _p]),
}


class HotPathError(RuntimeError):
    """A call into libb200hot.so failed (message from hp_last_error)."""


_LIB = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise HotPathError(
            f"{p} not found: build it with `python -m paper_2504_19516_b200.build` "
            "(there is no CPU fallback for the hot path)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().hp_last_error().decode(errors="replace")
        if rc == -1:
            raise InvalidArgumentError(f"{what}: {msg}")
        raise HotPathError(f"{what} failed ({rc}): {msg}")


def wave_stats(g: int, b: int, n: int) -> tuple[int, int, float]:
    w, t, idle = _i64(), _i64(), C.c_double()
    check(load().hp_wave_stats(g, b, n, C.byref(w), C.byref(t), C.byref(idle)), "hp_wave_stats")
    return w.value, t.value, idle.value


# --------------------------------------------------------------- torch glue
def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch

    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def device_sms(device: int = 0) -> int:
    n = _i()
    check(load().hp_device_sms(device, C.byref(n)), "hp_device_sms")
    return n.value


def rmsnorm(x, weight, out, eps: float, max_ctas: int, stream=None) -> None:
    rows, cols = x.shape
    check(load().hp_rmsnorm(_ptr(x), x.stride(0), _ptr(weight), _ptr(out), out.stride(0), rows, cols,
                            eps, max_ctas, _stream(stream)), "hp_rmsnorm")


def tile_weight(w, stream=None):
    """Row-major [N, K] bf16 weight -> the tiled, pre-swizzled layout the GEMMs
    stream with bulk copies (same shape/size; opaque element order)."""
    import torch

    N, K = w.shape
    out = torch.empty_like(w, memory_format=torch.contiguous_format)
    check(load().hp_tile_weight(_ptr(w), w.stride(0), _ptr(out), N, K, _stream(stream)), "hp_tile_weight")
    return out


def gemm(x, w, y, epilogue: int = EPI_STORE, resid=None, max_ctas: int = 148, stream=None) -> None:
    """Y = epi(X . W^T) with `w` from tile_weight()."""
    T, K = x.shape
    N = w.shape[0]
    check(load().hp_gemm(_ptr(x), x.stride(0), _ptr(w), w.stride(0), _ptr(y), y.stride(0),
                         _ptr(resid), resid.stride(0) if resid is not None else 0, T, N, K,
                         epilogue, max_ctas, _stream(stream)), "hp_gemm")


def gemm_traced(x, w, y, cta_times, epilogue: int = EPI_STORE, resid=None, max_ctas: int = 148,
                stream=None) -> None:
    """hp_gemm that also records per-CTA {smid, start_ns, end_ns} (int64 [grid, 3])."""
    T, K = x.shape
    N = w.shape[0]
    check(load().hp_gemm_traced(_ptr(x), x.stride(0), _ptr(w), w.stride(0), _ptr(y), y.stride(0),
                                _ptr(resid), resid.stride(0) if resid is not None else 0, T, N, K,
                                epilogue, max_ctas, _ptr(cta_times), _stream(stream)), "hp_gemm_traced")


def gemm_tiles(T: int, N: int) -> int:
    return load().hp_gemm_tiles(T, N)


def gemm_swap_ws_bytes(T: int, N: int, K: int, max_ctas: int) -> int:
    return load().hp_gemm_swap_ws_bytes(T, N, K, max_ctas)


def gemm_swap(x, w, y, ws, counters, epilogue: int = EPI_STORE, resid=None,
              max_ctas: int = 148, stream=None) -> None:
    """Decode GEMM (T <= 256), `w` from tile_weight()."""
    T, K = x.shape
    N = w.shape[0]
    check(load().hp_gemm_swap(_ptr(x), x.stride(0), _ptr(w), w.stride(0), _ptr(y), y.stride(0),
                              _ptr(resid), resid.stride(0) if resid is not None else 0, T, N, K,
                              epilogue, _ptr(ws), 0 if ws is None else ws.numel() * ws.element_size(),
                              _ptr(counters), 0 if counters is None else counters.numel(), max_ctas,
                              _stream(stream)), "hp_gemm_swap")


def gemm_swap_qkv_rope(x, w, y, Hq: int, Hkv: int, d: int, positions, cos_sin, slots, kcache, vcache,
                       page: int, ws, counters, max_ctas: int = 148, stream=None) -> None:
    """Decode QKV GEMM (T <= 256) with RoPE and the paged K/V write in the
    epilogue: gemm_swap(..., EPI_STORE) + rope_kv_write in one launch."""
    T, K = x.shape
    check(load().hp_gemm_swap_qkv_rope(_ptr(x), x.stride(0), _ptr(w), w.stride(0), _ptr(y), y.stride(0), T, Hq,
                                       Hkv, d, K, _ptr(positions), _ptr(cos_sin), _ptr(slots), _ptr(kcache),
                                       _ptr(vcache), page, _ptr(ws),
                                       0 if ws is None else ws.numel() * ws.element_size(), _ptr(counters),
                                       0 if counters is None else counters.numel(), max_ctas, _stream(stream)),
          "hp_gemm_swap_qkv_rope")


def peer_tiles(T: int, N: int) -> int:
    n = load().hp_peer_tiles(T, N)
    if n < 0:
        raise InvalidArgumentError(f"peer_tiles: bad shape T={T} N={N}")
    return n


def gemm_swap_peer(x, w, peer_recv, recv_half: int, peer_flags, flags_half: int, world: int, rank: int,
                   epoch: int, epoch_dev, ws, counters, max_ctas: int = 148, stream=None,
                   two_shot: bool = False) -> None:
    """Row-parallel decode GEMM whose epilogue scatters this rank's partial
    into every rank's receive buffer; peer_recv / peer_flags: ctypes arrays
    of `world` base device pointers (see include/hp.h hp_gemm_swap_peer);
    epoch_dev: device int tensor (device epochs) or None (host `epoch`)."""
    T, K = x.shape
    N = w.shape[0]
    check(load().hp_gemm_swap_peer(_ptr(x), x.stride(0), _ptr(w), w.stride(0), T, N, K, peer_recv, recv_half,
                                   peer_flags, flags_half, world, rank, epoch, _ptr(epoch_dev), int(two_shot),
                                   _ptr(ws),
                                   ws.numel() * ws.element_size(), _ptr(counters), counters.numel(), max_ctas,
                                   _stream(stream)), "hp_gemm_swap_peer")


def peer_reduce(recv_ptr: int, recv_half: int, flags_ptr: int, flags_half: int, world: int, T: int, N: int,
                epoch: int, out, resid=None, epoch_dev=None, done=None, stream=None) -> None:
    check(load().hp_peer_reduce(recv_ptr, recv_half, flags_ptr, flags_half, world, T, N, epoch, _ptr(epoch_dev),
                                _ptr(done), _ptr(resid), resid.stride(0) if resid is not None else 0, _ptr(out),
                                out.stride(0), _stream(stream)), "hp_peer_reduce")


def peer_rs(recv_ptr: int, recv_half: int, flags_ptr: int, flags_half: int, peer_gather, gather_half: int,
            peer_gflags, gflags_half: int, world: int, rank: int, T: int, N: int, epoch: int, epoch_dev=None,
            resid=None, stream=None) -> None:
    check(load().hp_peer_rs(recv_ptr, recv_half, flags_ptr, flags_half, peer_gather, gather_half, peer_gflags,
                            gflags_half, world, rank, T, N, epoch, _ptr(epoch_dev), _ptr(resid),
                            resid.stride(0) if resid is not None else 0, _stream(stream)), "hp_peer_rs")


def peer_ag(gather_ptr: int, gather_half: int, gflags_ptr: int, gflags_half: int, T: int, N: int, epoch: int,
            out, epoch_dev=None, done=None, stream=None) -> None:
    check(load().hp_peer_ag(gather_ptr, gather_half, gflags_ptr, gflags_half, T, N, epoch, _ptr(epoch_dev),
                            _ptr(done), _ptr(out), out.stride(0), _stream(stream)), "hp_peer_ag")


def ipc_handle(t) -> tuple[bytes, int]:
    """(handle of t's allocation block, t's byte offset inside it)."""
    buf = C.create_string_buffer(IPC_HANDLE_BYTES)
    off = C.c_size_t()
    check(load().hp_ipc_handle(_ptr(t), buf, C.byref(off)), "hp_ipc_handle")
    return buf.raw, off.value


def ipc_open(handle: bytes) -> int:
    """Map a peer's block; returns its base pointer in this process."""
    p = C.c_void_p()
    check(load().hp_ipc_open(C.create_string_buffer(handle, IPC_HANDLE_BYTES), C.byref(p)), "hp_ipc_open")
    return p.value


def ipc_close(ptr: int) -> None:
    check(load().hp_ipc_close(ptr), "hp_ipc_close")


def rope_kv_write(qkv, Hq: int, Hkv: int, d: int, positions, cos_sin, slots, kcache, vcache,
                  page: int, max_ctas: int = 148, stream=None) -> None:
    T = qkv.shape[0]
    check(load().hp_rope_kv_write(_ptr(qkv), qkv.stride(0), T, Hq, Hkv, d, _ptr(positions),
                                  _ptr(cos_sin), _ptr(slots), _ptr(kcache), _ptr(vcache), page,
                                  max_ctas, _stream(stream)), "hp_rope_kv_write")


def prefill_attn(q, k, v, o, cu_seqlens, nseq: int, max_seqlen: int, Hq: int, Hkv: int, d: int,
                 scale: float, max_ctas: int = 148, stream=None) -> None:
    check(load().hp_prefill_attn(_ptr(q), q.stride(0), _ptr(k), k.stride(0), _ptr(v), v.stride(0),
                                 _ptr(o), o.stride(0), _ptr(cu_seqlens), nseq, q.shape[0], max_seqlen, Hq, Hkv,
                                 d, scale, max_ctas, _stream(stream)), "hp_prefill_attn")


def gemm_qkv_rope(x, w, y, Hq: int, Hkv: int, d: int, positions, cos_sin, slots, kcache, vcache,
                  page: int, max_ctas: int = 148, stream=None) -> None:
    """Fused prefill QKV GEMM + RoPE + paged K/V write (hp_gemm_qkv_rope)."""
    check(load().hp_gemm_qkv_rope(_ptr(x), x.stride(0), _ptr(w), x.shape[1], _ptr(y), y.stride(0), x.shape[0], Hq,
                                  Hkv, d, x.shape[1], _ptr(positions), _ptr(cos_sin), _ptr(slots), _ptr(kcache),
                                  _ptr(vcache), page, max_ctas, _stream(stream)), "hp_gemm_qkv_rope")


def gemm_plan(T: int, N: int, K: int, max_ctas: int) -> tuple[int, int, int]:
    """(tile width, tile count, CTAs per tile) hp_gemm uses on a
    `max_ctas`-SM partition; without a stream-K tail (gemm_tail_tiles == 0)
    its persistent grid runs wave_stats(tiles, 1, max_ctas // ctas_per_tile)
    rounds."""
    bn, tiles, cpt, tail = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(load().hp_gemm_plan(T, N, K, max_ctas, C.byref(bn), C.byref(tiles), C.byref(cpt), C.byref(tail)),
          "hp_gemm_plan")
    return bn.value, tiles.value, cpt.value


def gemm_tail_tiles(T: int, N: int, K: int, max_ctas: int) -> int:
    """Tiles hp_gemm's stream-K tail splits over every pair (0: plain rounds)."""
    bn, tiles, cpt, tail = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(load().hp_gemm_plan(T, N, K, max_ctas, C.byref(bn), C.byref(tiles), C.byref(cpt), C.byref(tail)),
          "hp_gemm_plan")
    return tail.value


def prefill_attn_paged(q, kcache, vcache, block_table, cu_seqlens, prior_lens, nseq: int, max_seqlen: int,
                       o, Hq: int, Hkv: int, d: int, page: int, scale: float, max_ctas: int = 148,
                       stream=None) -> None:
    """Chunked-prefill attention: new tokens (rows of q) over cached prefix + span."""
    check(load().hp_prefill_attn_paged(_ptr(q), q.stride(0), _ptr(kcache), _ptr(vcache), _ptr(block_table),
                                       block_table.shape[1], _ptr(cu_seqlens), _ptr(prior_lens), nseq,
                                       q.shape[0], max_seqlen, _ptr(o), o.stride(0), Hq, Hkv, d, page,
                                       kcache.shape[0], scale, max_ctas, _stream(stream)),
          "hp_prefill_attn_paged")


def decode_attn_launches(B: int, Hq: int, Hkv: int, d: int, max_pages: int, page: int, max_ctas: int) -> int:
    return load().hp_decode_attn_launches(B, Hq, Hkv, d, max_pages, page, max_ctas)


def decode_attn_ws_bytes(B: int, Hq: int, d: int, max_splits: int) -> int:
    return load().hp_decode_attn_ws_bytes(B, Hq, d, max_splits)


def decode_attn(q, kcache, vcache, block_table, ctx_lens, out, Hq: int, Hkv: int, d: int,
                page: int, scale: float, ws=None, max_ctas: int = 148, stream=None) -> None:
    B = q.shape[0]
    check(load().hp_decode_attn(_ptr(q), q.stride(0), _ptr(kcache), _ptr(vcache), _ptr(block_table),
                                block_table.shape[1], _ptr(ctx_lens), _ptr(out), out.stride(0), B, Hq,
                                Hkv, d, page, kcache.shape[0], scale, _ptr(ws),
                                0 if ws is None else ws.numel() * ws.element_size(), max_ctas,
                                _stream(stream)), "hp_decode_attn")


def copy_rows(src, dst, max_ctas: int = 148, stream=None) -> None:
    """dst[:] = src for 2-D tensors of equal shape/dtype (either may be pinned
    host memory, read or written through UVA by the kernel)."""
    if src.shape != dst.shape or src.dtype != dst.dtype or src.dim() != 2:
        raise InvalidArgumentError("copy_rows: src/dst must be 2-D with equal shape and dtype")
    es = src.element_size()
    check(load().hp_copy_rows(_ptr(src), src.stride(0) * es, _ptr(dst), dst.stride(0) * es, src.shape[0],
                              src.shape[1] * es, max_ctas, _stream(stream)), "hp_copy_rows")


_SIDE: dict = {}


def hold(stream, cycles: int) -> None:
    """Delay the work queued next on `stream` by ~`cycles` GPU clocks (so a
    burst of host launches is queued before any of it runs).  The spin
    kernel runs on a primary-context side stream that `stream` then waits on:
    torch's spin kernel launched straight into a green-context stream is the
    one kernel ncu fails to prepare for profiling."""
    import torch

    dev = stream.device
    side = _SIDE.get(dev)
    if side is None:
        side = _SIDE[dev] = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        torch.cuda._sleep(cycles)
    stream.wait_stream(side)


def set_trace(kind: int, buf) -> None:
    check(load().hp_set_trace(kind, _ptr(buf)), "hp_set_trace")


def gemm_tail_reserve(stream) -> None:
    """Allocate the stream-K fix-up workspace of `stream` (a torch stream or
    raw handle) now rather than on its first tail GEMM."""
    check(load().hp_gemm_tail_reserve(_stream(stream)), "hp_gemm_tail_reserve")


def set_gemm_tail(mode: int) -> None:
    """Stream-K tail of the prefill CTA-pair GEMM: 1 on, 0 off (plain
    persistent rounds, the grid wave_stats describes), -1 the HP_GEMM_TAIL
    environment default (on)."""
    check(load().hp_set_gemm_tail(mode), "hp_set_gemm_tail")


TRACE_CTAS = 2


def arm_cta_trace(buf) -> None:
    """The next prefill GEMM / attention launch records per-CTA {smid,
    start_ns, end_ns} into `buf` (uint64/int64 [grid, 3]); one-shot."""
    set_trace(TRACE_CTAS, buf)


def cta_idle(times, sms: int) -> tuple[float, float, int]:
    """(idle fraction, span s, CTAs) of one traced launch on an `sms`-SM
    partition: 1 - sum(CTA busy) / (sms x kernel span) -- config 3's
    measured idle, against wave_stats(units, 1, slots) (perf_model.py:157-169)."""
    t = times.cpu()
    t = t[t[:, 2] > 0]
    start, end = t[:, 1], t[:, 2]
    span = float(end.max() - start.min())
    busy = float((end - start).sum())
    return 1.0 - busy / (sms * span), span * 1e-9, int(t.shape[0])


def membw(src, ctas: int, method: int, out, stream=None) -> None:
    check(load().hp_membw(_ptr(src), src.numel() * src.element_size(), ctas, method, _ptr(out),
                          _stream(stream)), "hp_membw")


def _kv_chunk_index(x7):
    """Gather index swapping 16-byte chunk c of token row r with c ^ (r & 7)
    over a [nb, H, tiles, halves, 64 rows, 8 chunks, 8] view."""
    import torch

    r = torch.arange(64, device=x7.device)
    c = torch.arange(8, device=x7.device)
    src = c[None, :] ^ (r[:, None] & 7)
    return src[None, None, None, None, :, :, None].expand(*x7.shape)


def kv_pack(x):
    """Logical K or V cache [blocks, Hkv, page, d] -> the device page layout
    ([blocks, Hkv, page/64, d/64, 64, 64]: 64-token tiles, each a contiguous
    run of 64-dim halves with 128B-swizzled chunks), returned as a tensor of
    the same shape whose memory is in device order."""
    import torch

    nb, H, P, d = x.shape
    v = x.reshape(nb, H, P // 64, 64, d // 64, 8, 8).permute(0, 1, 2, 4, 3, 5, 6)
    return torch.gather(v, 5, _kv_chunk_index(v)).contiguous().view(nb, H, P, d)


def kv_unpack(y):
    """Inverse of kv_pack."""
    import torch

    nb, H, P, d = y.shape
    v = y.reshape(nb, H, P // 64, d // 64, 64, 8, 8)
    v = torch.gather(v, 5, _kv_chunk_index(v))
    return v.permute(0, 1, 2, 4, 3, 5, 6).contiguous().view(nb, H, P, d)


def probe(out, ctas: int, threads: int = 128, spin_ns: int = 20000, stream=None) -> None:
    check(load().hp_probe(ctas, threads, spin_ns, _ptr(out), _stream(stream)), "hp_probe")


class Partition:
    """A green-context SM split: `decode_sms` SMs for decode, the rest for prefill.

    Realises the reference's partition masks (engine.py:440-452) on hardware;
    `stream(phase)` returns a torch ExternalStream confined to that side.
    """

    def __init__(self, decode_sms: int, device: int = 0):
        h = _p()
        check(load().hp_partition_create(device, decode_sms, C.byref(h)), "hp_partition_create")
        self._h = h
        self.device = device
        self.sms = {}
        self._streams = {}
        for phase in (0, 1):
            n = _i()
            check(load().hp_partition_sms(h, phase, C.byref(n)), "hp_partition_sms")
            self.sms[phase] = n.value
            s = _p()
            check(load().hp_partition_stream(h, phase, C.byref(s)), "hp_partition_stream")
            self._streams[phase] = s.value

    @property
    def prefill_sms(self) -> int:
        return self.sms[0]

    @property
    def decode_sms(self) -> int:
        return self.sms[1]

    def raw_stream(self, phase: int) -> int:
        return self._streams[phase]

    def stream(self, phase: int):
        import torch

        return torch.cuda.ExternalStream(self._streams[phase], device=torch.device("cuda", self.device))

    def close(self) -> None:
        if self._h is not None:
            load().hp_partition_destroy(self._h)
            self._h = None

    # No __del__: destroying a green context while torch still holds events or
    # cached streams on it aborts at interpreter exit; partitions live for the
    # process unless close() is called explicitly.
