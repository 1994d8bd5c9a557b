"""SM partition pool: the hardware side of `_request_partition` /
`_apply_partitions` (reference engine.py:440-467).

The reference models an SM-mask change as a `reconfig_s` delay
(engine.py:132).  On the B200 a split (pm prefill SMs, dm decode SMs) is a
pre-created green-context pair whose streams confine every kernel launched
into them to that side's SMs; "reconfiguring" is choosing which pair's
streams the next launches go to (no driver call on the hot path).

Green contexts need SM groups in multiples of 8 on CC >= 9 (cuda.h,
cuDevSmResourceSplitByCount), so decode shares live on the 8-grid and the
prefill side takes the remainder (148 = 18*8 + 4).  A phase granted all N
SMs runs on a plain full-device stream (one per phase, so the two phases
still overlap -- the reference's `nopartition` / transition-window
behaviour, engine.py:457-466, scheduler.py:398-409).
"""

from __future__ import annotations

import torch

from . import lib

PREFILL, DECODE = 0, 1


class PhaseStreams:
    """Where one phase's next launches go: a raw cudaStream_t plus the SM
    count that sizes its persistent grids."""

    __slots__ = ("stream", "sms", "torch_stream")

    def __init__(self, stream: int, sms: int, torch_stream):
        self.stream = stream
        self.sms = sms
        self.torch_stream = torch_stream


class _GridOnlyPartition:
    """HP_NO_GREEN=1 (profiling only): plain streams with the split's SM
    counts as grid sizes and no confinement.  ncu cannot prepare kernels
    launched into green-context streams on this driver, so the launch list
    is captured in this mode; every kernel keeps the grid it has in the
    real co-run, and ncu serialises launches anyway."""

    def __init__(self, decode_sms: int, device: int, n: int):
        import torch

        self.sms = {0: n - decode_sms, 1: decode_sms}
        self._streams = {ph: torch.cuda.Stream(device=device) for ph in (0, 1)}

    def raw_stream(self, phase: int) -> int:
        return self._streams[phase].cuda_stream

    def stream(self, phase: int):
        return self._streams[phase]

    def close(self) -> None:
        pass


class PartitionPool:
    def __init__(self, device: int = 0, granularity: int = 8):
        import os

        self.device = device
        self.grid_only = os.environ.get("HP_NO_GREEN") == "1"
        self.n = lib.device_sms(device)
        self.granularity = granularity
        self._parts: dict[int, lib.Partition] = {}
        self._full = {PREFILL: torch.cuda.Stream(device=device), DECODE: torch.cuda.Stream(device=device)}
        # prefill streams get their GEMM stream-K workspace at creation, not
        # on a first tail GEMM in the middle of a timed / served run
        lib.gemm_tail_reserve(self._full[PREFILL])

    def realizable_decode_sms(self, dm: int) -> int:
        """Round a requested decode share up to the green-context grid."""
        g = self.granularity
        dm = max(g, -(-dm // g) * g)
        return min(dm, (self.n - 1) // g * g)

    def partition(self, dm: int) -> lib.Partition:
        dm = self.realizable_decode_sms(dm)
        part = self._parts.get(dm)
        if part is None:
            part = _GridOnlyPartition(dm, self.device, self.n) if self.grid_only else lib.Partition(dm, self.device)
            lib.gemm_tail_reserve(part.raw_stream(PREFILL))
            self._parts[dm] = part
        return part

    def full(self, phase: int) -> PhaseStreams:
        s = self._full[phase]
        return PhaseStreams(s.cuda_stream, self.n, s)

    def phase(self, phase: int, share: int) -> PhaseStreams:
        """Streams for `phase` holding `share` SMs (the other phase holds the rest)."""
        if share >= self.n:
            return self.full(phase)
        if share < 1:
            raise ValueError("phase has no SMs")
        dm = share if phase == DECODE else self.n - share
        part = self.partition(dm)
        return PhaseStreams(part.raw_stream(phase), part.sms[phase], part.stream(phase))

    def split(self, pm: int, dm: int) -> tuple[PhaseStreams | None, PhaseStreams | None]:
        """Prefill/decode streams for the decision (pm, dm).  pm + dm <= N uses
        one green-context pair; pm + dm > N (transition handoff) keeps prefill
        in its partition and runs decode device-wide."""
        ps = ds = None
        if pm >= 1 and dm >= 1 and pm + dm <= self.n and pm < self.n and dm < self.n:
            part = self.partition(dm)
            ps = PhaseStreams(part.raw_stream(PREFILL), part.sms[PREFILL], part.stream(PREFILL))
            ds = PhaseStreams(part.raw_stream(DECODE), part.sms[DECODE], part.stream(DECODE))
            return ps, ds
        if pm >= 1:
            ps = self.phase(PREFILL, pm)
        if dm >= 1:
            ds = self.phase(DECODE, dm)
        return ps, ds

    def warm(self, shares=None) -> None:
        """Create every decode share on the grid up front (avoid first-use cost)."""
        for dm in shares or range(self.granularity, self.n, self.granularity):
            self.partition(dm)

    def close(self) -> None:
        for p in self._parts.values():
            p.close()
        self._parts.clear()
