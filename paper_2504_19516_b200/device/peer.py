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
step without a host barrier (include/hp.h, hp_gemm_swap_peer).  With
`device_epoch=True` the epoch lives in device memory (read by the GEMM and the
reduce, advanced by the reduce's last block), so a captured CUDA graph of the
layer replays correctly; the default host epochs suit eager launches.

`two_shot=True` switches to the bandwidth-optimal form for large batches:
the GEMM sends each 128-feature tile only to its owner rank (mt % world),
the owner reduces it and broadcasts the result into every rank's gather
buffer (hp_peer_rs), and every rank copies the gathered tiles out
(hp_peer_ag): 2 (world-1)/world of the message per rank instead of
(world-1) x, one extra hop.  Extra symmetric buffers:
    gather  bf16 [2][T_max][N]             gflags int [2][ceil(T_max/16)][N/128]

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
                 flags: torch.Tensor | None, peer_recv: list[int], peer_flags: list[int], device,
                 device_epoch: bool = False, gather=None, peer_gather=None, peer_gflags=None):
        if not 1 <= world <= lib.MAX_PEERS:
            raise ValueError(f"world {world} outside [1, {lib.MAX_PEERS}]")
        if not 1 <= T_max <= 256 or N % 128:
            raise ValueError("fused all-reduce: T_max in [1, 256], N a multiple of 128")
        self.world, self.rank, self.T_max, self.N = world, rank, T_max, N
        self.recv, self.flags = recv, flags          # this rank's own buffers (kept alive)
        self.dev = device
        self.half_recv = world * T_max * N           # elements (bf16)
        self.half_flags = world * lib.peer_tiles(T_max, N)  # elements (int32)
        self._peer_recv = peer_recv
        self._peer_flags = peer_flags
        self._rv = (C.c_void_p * world)(*peer_recv)
        self._fl = (C.c_void_p * world)(*peer_flags)
        self._opened: list[int] = []
        self.epoch = 0
        self._ws = None
        self._ws_retired: list = []  # outgrown workspaces, kept alive for captured graphs
        # device epoch + the reduce's block counter (both start at zero)
        self.epoch_dev = torch.zeros(2, dtype=torch.int32, device=device) if device_epoch else None
        self.two_shot = peer_gather is not None
        if self.two_shot:
            self.gather = gather  # this rank's (gather, gflags), kept alive
            self.half_gather = T_max * N
            self.half_gflags = -(-T_max // 16) * (N // 128)
            self._peer_gather, self._peer_gflags = peer_gather, peer_gflags
            self._gv = (C.c_void_p * world)(*peer_gather)
            self._gf = (C.c_void_p * world)(*peer_gflags)

    # ---------------------------------------------------------- construction
    @staticmethod
    def _alloc(world, T_max, N, device):
        recv = torch.empty(2 * world * T_max * N, dtype=torch.bfloat16, device=device)
        flags = torch.zeros(2 * world * lib.peer_tiles(T_max, N), dtype=torch.int32, device=device)
        return recv, flags

    @staticmethod
    def _alloc_gather(T_max, N, device):
        gather = torch.empty(2 * T_max * N, dtype=torch.bfloat16, device=device)
        gflags = torch.zeros(2 * -(-T_max // 16) * (N // 128), dtype=torch.int32, device=device)
        return gather, gflags

    @classmethod
    def local_group(cls, world: int, T_max: int, N: int, device=None, device_epoch: bool = False,
                    two_shot: bool = False) -> list["PeerAllReduce"]:
        """`world` ranks emulated in one process: every rank's buffers live on
        this GPU and the 'peer' pointers are plain device pointers."""
        device = device or torch.device("cuda", torch.cuda.current_device())
        bufs = [cls._alloc(world, T_max, N, device) for _ in range(world)]
        pr = [r.data_ptr() for r, _ in bufs]
        pf = [f.data_ptr() for _, f in bufs]
        gat = [cls._alloc_gather(T_max, N, device) for _ in range(world)] if two_shot else None
        pg = [g.data_ptr() for g, _ in gat] if two_shot else None
        pgf = [f.data_ptr() for _, f in gat] if two_shot else None
        ranks = [cls(world, q, T_max, N, bufs[q][0], bufs[q][1], pr, pf, device, device_epoch,
                     gat[q] if two_shot else None, pg, pgf) for q in range(world)]
        for r in ranks:  # every rank's buffers stay alive as long as any rank's view does
            r._group_buffers = (bufs, gat)
        return ranks

    @classmethod
    def create(cls, group, T_max: int, N: int, device=None, device_epoch: bool = False,
               two_shot: bool = False) -> "PeerAllReduce":
        """One rank of a multi-process TP group: allocate this rank's buffers,
        exchange CUDA IPC handles over `group`, map every peer's buffers."""
        import os

        import torch.distributed as dist

        conf = os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "") + "," + os.environ.get("PYTORCH_ALLOC_CONF", "")
        if "expandable_segments:true" in conf.replace(" ", "").lower():
            # expandable segments are cuMemCreate (VMM) allocations, which
            # legacy cudaIpcGetMemHandle cannot export
            raise RuntimeError("PeerAllReduce.create: CUDA IPC of caching-allocator blocks does not work "
                               "with PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True; unset it")
        device = device or torch.device("cuda", torch.cuda.current_device())
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        recv, flags = cls._alloc(world, T_max, N, device)
        own = [recv, flags]
        gat = cls._alloc_gather(T_max, N, device) if two_shot else None
        if two_shot:
            own += list(gat)
        torch.cuda.synchronize(device)
        mine = tuple(lib.ipc_handle(t) for t in own)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        ptrs = [[] for _ in own]  # per buffer kind: one pointer per rank
        opened = {}
        for q in range(world):
            for k, (h, off) in enumerate(allh[q]):
                if q == rank:
                    ptrs[k].append(own[k].data_ptr())
                    continue
                if h not in opened:  # buffers may share one allocation block
                    opened[h] = lib.ipc_open(h)
                ptrs[k].append(opened[h] + off)
        pr, pf = ptrs[0], ptrs[1]
        self = cls(world, rank, T_max, N, recv, flags, pr, pf, device, device_epoch, gat,
                   ptrs[2] if two_shot else None, ptrs[3] if two_shot else None)
        self._opened = list(opened.values())
        dist.barrier(group=group)
        return self

    def close(self) -> None:
        for p in self._opened:
            lib.ipc_close(p)
        self._opened = []

    # ------------------------------------------------------------------ call
    def workspace(self, K: int, max_ctas: int):
        """Stream-K workspace + arrival counters for a K-deep GEMM.  Sized for
        148 CTAs (any partition) and grown only for a deeper K; a replaced
        workspace is retained, never freed, because CUDA graphs captured
        earlier (e.g. on a smaller partition) keep its pointers.  A new
        workspace's zeroed counters are made visible to every stream before
        first use (the GEMM may run on a green-context stream)."""
        nb = lib.gemm_swap_ws_bytes(256, self.N, K, max(max_ctas, 148))
        if self._ws is None or self._ws[0].numel() * 4 < nb:
            if self._ws is not None:
                self._ws_retired.append(self._ws)
            self._ws = (torch.empty(nb // 4 + 1, dtype=torch.float32, device=self.dev),
                        torch.zeros(self.N // 128 * 8, dtype=torch.int32, device=self.dev))
            torch.cuda.synchronize(self.dev)
        return self._ws

    def gemm(self, x, w, epoch: int, max_ctas: int = 148, stream=None) -> None:
        """Epilogue half: this rank's partial x @ w^T scattered to every rank."""
        T = x.shape[0]
        if T > self.T_max or w.shape[0] != self.N:
            raise ValueError(f"fused all-reduce sized for T <= {self.T_max}, N = {self.N}")
        ws, cnt = self.workspace(x.shape[1], max_ctas)
        lib.gemm_swap_peer(x, w, C.cast(self._rv, C.c_void_p), self.half_recv, C.cast(self._fl, C.c_void_p),
                           self.half_flags, self.world, self.rank, epoch, self._edev(), ws, cnt,
                           max_ctas=max_ctas, stream=stream, two_shot=self.two_shot)

    def reduce(self, out, epoch: int, resid=None, stream=None) -> None:
        """Receive half: out = sum over ranks of the partials (+ resid).
        Two-shot: reduce_scatter() then all_gather() (separate launches)."""
        if self.two_shot:
            self.reduce_scatter(out.shape[0], epoch, resid, stream)
            self.all_gather(out, epoch, stream)
            return
        T = out.shape[0]
        e = self._edev()
        lib.peer_reduce(self._peer_recv[self.rank], self.half_recv, self._peer_flags[self.rank], self.half_flags,
                        self.world, T, self.N, epoch, out, resid=resid, epoch_dev=e,
                        done=None if e is None else self.epoch_dev[1:], stream=stream)

    def reduce_scatter(self, T: int, epoch: int, resid=None, stream=None) -> None:
        lib.peer_rs(self._peer_recv[self.rank], self.half_recv, self._peer_flags[self.rank], self.half_flags,
                    C.cast(self._gv, C.c_void_p), self.half_gather, C.cast(self._gf, C.c_void_p), self.half_gflags,
                    self.world, self.rank, T, self.N, epoch, epoch_dev=self._edev(), resid=resid, stream=stream)

    def all_gather(self, out, epoch: int, stream=None) -> None:
        e = self._edev()
        lib.peer_ag(self._peer_gather[self.rank], self.half_gather, self._peer_gflags[self.rank], self.half_gflags,
                    out.shape[0], self.N, epoch, out, epoch_dev=e, done=None if e is None else self.epoch_dev[1:],
                    stream=stream)

    def _edev(self):
        return None if self.epoch_dev is None else self.epoch_dev[:1]

    def linear(self, x, w, out, resid=None, max_ctas: int = 148, stream=None) -> None:
        """out = all_reduce(x @ w^T) + resid, fused (one process per rank)."""
        self.epoch += 1
        self.gemm(x, w, self.epoch, max_ctas, stream)
        self.reduce(out, self.epoch, resid, stream)
