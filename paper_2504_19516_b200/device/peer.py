"""Fused row-parallel GEMM + all-reduce for tensor-parallel decode
(BASELINE config 5).

The unfused TP layer (tp.py) runs o_proj / mlp_down as a GEMM that writes a
bf16 partial, then an NCCL all-reduce of T x hidden.  For decode (T <= 256)
the message is small (<= 4 MiB at hidden 8192) and latency-bound, so here the
GEMM itself does the exchange: the swap-AB stream-K kernel's epilogue stores
each finished 128-feature x BN-token partial tile straight into slot `rank`
of every rank's receive buffer over NVLink peer memory and raises a per-tile
flag; a small reduce kernel on each rank waits for the tile's `world` flags
and writes sum + residual.  The transfer of one tile overlaps the MMA of the
next and there is no separate collective launch.

Symmetric memory (one set per rank, mapped by every peer with CUDA IPC):
    recv  bf16 [2][world][T_max][N]     half (epoch & 1) per call
    flags int  [2][world][tiles_max]    zero at allocation; values = epoch
Epochs start at 1 and advance by one per call on every rank, so ranks stay in
step without a host barrier (include/hp.h, hp_gemm_swap_peer).

`PeerAllReduce.local_group` builds `world` instances inside ONE process on
one GPU (all buffers local): the same kernels and flag protocol, used by the
single-GPU tests and to measure the epilogue's cost; `PeerAllReduce.create`
is the real multi-process constructor (one process per GPU, handles
exchanged through a torch.distributed group).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import lib


class PeerAllReduce:
    def __init__(self, world: int, rank: int, T_max: int, N: int, recv: torch.Tensor | None,
                 flags: torch.Tensor | None, peer_recv: list[int], peer_flags: list[int], device):
        if not 1 <= world <= lib.MAX_PEERS:
            raise ValueError(f"world {world} outside [1, {lib.MAX_PEERS}]")
        if not 1 <= T_max <= 256 or N % 128:
            raise ValueError("fused all-reduce: T_max in [1, 256], N a multiple of 128")
        self.world, self.rank, self.T_max, self.N = world, rank, T_max, N
        self.recv, self.flags = recv, flags          # this rank's own buffers (kept alive)
        self.dev = device
        self.half_recv = world * T_max * N * 2       # bytes
        self.half_flags = world * lib.peer_tiles(T_max, N) * 4
        self._peer_recv = peer_recv
        self._peer_flags = peer_flags
        self._ptr_arrays = {}
        self._opened: list[int] = []
        self.epoch = 0
        self._ws = None

    # ---------------------------------------------------------- construction
    @staticmethod
    def _alloc(world, T_max, N, device):
        recv = torch.empty(2 * world * T_max * N, dtype=torch.bfloat16, device=device)
        flags = torch.zeros(2 * world * lib.peer_tiles(T_max, N), dtype=torch.int32, device=device)
        return recv, flags

    @classmethod
    def local_group(cls, world: int, T_max: int, N: int, device=None) -> list["PeerAllReduce"]:
        """`world` ranks emulated in one process: every rank's buffers live on
        this GPU and the 'peer' pointers are plain device pointers."""
        device = device or torch.device("cuda", torch.cuda.current_device())
        bufs = [cls._alloc(world, T_max, N, device) for _ in range(world)]
        pr = [r.data_ptr() for r, _ in bufs]
        pf = [f.data_ptr() for _, f in bufs]
        return [cls(world, q, T_max, N, bufs[q][0], bufs[q][1], pr, pf, device) for q in range(world)]

    @classmethod
    def create(cls, group, T_max: int, N: int, device=None) -> "PeerAllReduce":
        """One rank of a multi-process TP group: allocate this rank's buffers,
        exchange CUDA IPC handles over `group`, map every peer's buffers."""
        import torch.distributed as dist

        device = device or torch.device("cuda", torch.cuda.current_device())
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        recv, flags = cls._alloc(world, T_max, N, device)
        torch.cuda.synchronize(device)
        mine = (lib.ipc_handle(recv), lib.ipc_handle(flags))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        pr, pf, opened = [], [], {}
        for q in range(world):
            if q == rank:
                pr.append(recv.data_ptr())
                pf.append(flags.data_ptr())
                continue
            for (h, off), dst in zip(allh[q], (pr, pf)):
                if h not in opened:  # recv and flags may share one allocation block
                    opened[h] = lib.ipc_open(h)
                dst.append(opened[h] + off)
        self = cls(world, rank, T_max, N, recv, flags, pr, pf, device)
        self._opened = list(opened.values())
        dist.barrier(group=group)
        return self

    def close(self) -> None:
        for p in self._opened:
            lib.ipc_close(p)
        self._opened = []

    # ------------------------------------------------------------------ call
    def _arrays(self, half: int):
        a = self._ptr_arrays.get(half)
        if a is None:
            rv = (C.c_void_p * self.world)(*[p + half * self.half_recv for p in self._peer_recv])
            fl = (C.c_void_p * self.world)(*[p + half * self.half_flags for p in self._peer_flags])
            a = self._ptr_arrays[half] = (rv, fl)
        return a

    def workspace(self, K: int, max_ctas: int):
        nb = lib.gemm_swap_ws_bytes(256, self.N, K, max_ctas)
        if self._ws is None or self._ws[0].numel() * 4 < nb:
            self._ws = (torch.empty(nb // 4 + 1, dtype=torch.float32, device=self.dev),
                        torch.zeros(self.N // 128 * 8, dtype=torch.int32, device=self.dev))
        return self._ws

    def gemm(self, x, w, epoch: int, max_ctas: int = 148, stream=None) -> None:
        """Epilogue half: this rank's partial x @ w^T scattered to every rank."""
        T = x.shape[0]
        if T > self.T_max or w.shape[0] != self.N:
            raise ValueError(f"fused all-reduce sized for T <= {self.T_max}, N = {self.N}")
        rv, fl = self._arrays(epoch & 1)
        ws, cnt = self.workspace(x.shape[1], max_ctas)
        lib.gemm_swap_peer(x, w, C.cast(rv, C.c_void_p), C.cast(fl, C.c_void_p), self.world, self.rank, epoch,
                           ws, cnt, max_ctas=max_ctas, stream=stream)

    def reduce(self, out, epoch: int, resid=None, stream=None) -> None:
        """Receive half: out = sum over ranks of the partials (+ resid)."""
        T = out.shape[0]
        half = epoch & 1
        lib.peer_reduce(self._peer_recv[self.rank] + half * self.half_recv,
                        self._peer_flags[self.rank] + half * self.half_flags, self.world, T, self.N, epoch,
                        out, resid=resid, stream=stream)

    def linear(self, x, w, out, resid=None, max_ctas: int = 148, stream=None) -> None:
        """out = all_reduce(x @ w^T) + resid, fused (one process per rank)."""
        self.epoch += 1
        self.gemm(x, w, self.epoch, max_ctas, stream)
        self.reduce(out, self.epoch, resid, stream)
