"""Concurrent prefill/decode layer driver (the reference's `_launch_prefill` /
`_maybe_launch_decode` pair, engine.py:583-600 and 640-682, run for real).

A `CoRunner` holds one Llama layer in HBM with a prefill workload (one
sequence of T new tokens) and a decode workload (batch B over a paged KV
cache of context C).  It can execute, on the B200:

  * `isolated(phase, sms)`   one phase alone on a partition of `sms` SMs;
  * `corun(pm, dm, ...)`     prefill layers on a pm-SM green context while
                             decode layer-steps run on the dm-SM side;
  * `time_sliced(...)`       the non-partitioned baseline: the same work on
                             one full-GPU stream, prefill and decode
                             alternating (temporal sharing).

Decode steps are captured once per partition into a CUDA graph (one launch
per layer-step instead of nine or ten).  All times come from CUDA events recorded
on the launching streams.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass, field

import torch

from ..workload import ModelSpec
from . import lib
from .layer import (PAGE, DecodeScratch, DeviceLayer, KVCache, LayerWeights, PrefillScratch, mlp_width,
                    decode_slots)
from .partition import DECODE, PREFILL, PartitionPool, PhaseStreams


GROUPS = ("qkv", "attn", "o_proj", "mlp_up_gate", "mlp_down")


def _ev():
    return torch.cuda.Event(enable_timing=True)


def decode_schedule(steps: int, per_step) -> list[int]:
    """Decode layer-steps issued beside each of `steps` prefill layers:
    an int n (n each), a list (as given), or a float ratio r (Bresenham
    spread: r decode steps per prefill layer on average, at least 1 each --
    the decode side then runs continuously through the prefill layers)."""
    if isinstance(per_step, (list, tuple)):
        if len(per_step) != steps:
            raise ValueError("decode schedule length != steps")
        return [int(n) for n in per_step]
    if isinstance(per_step, int):
        return [per_step] * steps
    r = max(1.0, float(per_step))
    out, acc = [], 0.0
    for _ in range(steps):
        acc += r
        n = int(acc + 1e-9)
        out.append(n)
        acc -= n
    return out


@dataclass
class CoRunResult:
    pm: int
    dm: int
    steps: int
    decode_steps: int
    span_s: float
    prefill_tokens: int
    decode_tokens: int
    prefill_layer_s: list = field(default_factory=list)   # per prefill layer
    decode_layer_s: list = field(default_factory=list)    # per decode layer-step
    upgate_s: list = field(default_factory=list)          # dominant kernel launches
    group_s: dict = field(default_factory=dict)           # median seconds per prefill kernel group
    prefill_window_s: list = field(default_factory=list)  # (start, end) of each prefill layer from t0
    decode_window_s: list = field(default_factory=list)   # (start, end) of each decode layer-step

    def overlap_s(self) -> float:
        """Seconds during which a decode step ran while a prefill layer was
        running (the co-execution actually happened on the device)."""
        tot = 0.0
        for a0, a1 in self.prefill_window_s:
            for b0, b1 in self.decode_window_s:
                tot += max(0.0, min(a1, b1) - max(a0, b0))
        return tot

    def partition_idle(self, n: int) -> float:
        """SM idle fraction of the co-run: 1 - (pm * prefill busy + dm *
        decode busy) / (N * span) -- SM-time no partition had work for."""
        busy = self.pm * sum(self.prefill_layer_s) + self.dm * sum(self.decode_layer_s)
        return max(0.0, 1.0 - busy / (n * self.span_s))

    @property
    def tokens(self) -> int:
        return self.prefill_tokens + self.decode_tokens

    @property
    def tokens_per_s(self) -> float:
        return self.tokens / self.span_s

    def p50(self, xs) -> float:
        return statistics.median(xs) if xs else 0.0

    @property
    def ttft_layer_s(self) -> float:
        """Mean prefill progress per layer: completion of the last prefill
        layer / prefill layers (a prompt's TTFT is num_layers x this)."""
        return max(e for _, e in self.prefill_window_s) / self.steps

    @property
    def tpot_layer_s(self) -> float:
        """Mean time per decode layer-step: completion of the last decode
        step / decode steps (the mean inter-token time of a decoding
        request, per layer -- the paper's TPOT)."""
        return max(e for _, e in self.decode_window_s) / self.decode_steps


class CoRunner:
    def __init__(self, model: ModelSpec, prefill_tokens: int, decode_batch: int, decode_ctx: int,
                 device: int = 0, seed: int = 0, pool: PartitionPool | None = None,
                 weights: LayerWeights | None = None):
        self.model = model
        self.dev = torch.device("cuda", device)
        self.T = prefill_tokens
        self.B = decode_batch
        self.C = decode_ctx
        gen = torch.Generator(device="cpu")
        gen.manual_seed(seed)
        if weights is None:
            weights = LayerWeights.random(model, self.dev, gen)
        self.layer = DeviceLayer(model, weights, self.dev, max_pos=max(prefill_tokens, decode_ctx) + 1)
        self.pool = pool or PartitionPool(device)
        self.n = self.pool.n
        h = model.hidden
        bf = dict(dtype=torch.bfloat16, device=self.dev)
        # prefill workload
        self.px = torch.randn(self.T, h, generator=gen).to(**bf)
        self.py = torch.empty(self.T, h, **bf)
        self.psc = PrefillScratch(model, self.T + self.B, self.dev)  # hybrid batches: chunk + decode rows
        pblocks = -(-self.T // PAGE)
        self.pcache = KVCache(pblocks, model.num_kv_heads, model.head_dim, self.dev)
        self.p_cu = torch.tensor([0, self.T], dtype=torch.int32, device=self.dev)
        self.p_pos = torch.arange(self.T, dtype=torch.int32, device=self.dev)
        self.p_slots = torch.arange(self.T, dtype=torch.int32, device=self.dev)
        # decode workload: B sequences of context C over a shuffled block pool
        pages = -(-self.C // PAGE)
        nblk = self.B * pages
        # one page pool: decode sequences use the first B*pages blocks; the
        # chunked baseline's prefill sequence uses the last pblocks
        self.dcache = KVCache(nblk + pblocks, model.num_kv_heads, model.head_dim, self.dev)
        self.chunk_pages = torch.arange(nblk, nblk + pblocks, dtype=torch.int32, device=self.dev)[None]
        self.dcache.k.normal_(generator=None)
        self.dcache.v.normal_(generator=None)
        perm = torch.randperm(nblk, generator=gen).to(torch.int32)
        self.block_table = perm.view(self.B, pages).to(self.dev)
        self.ctx = torch.full((self.B,), self.C, dtype=torch.int32, device=self.dev)
        self.d_pos, self.d_slots = decode_slots(self.block_table, self.ctx)
        self.dx = torch.randn(self.B, h, generator=gen).to(**bf)
        self.dy = torch.empty(self.B, h, **bf)
        self.dsc = DecodeScratch(model, self.B, pages, self.dev, max_ctas=self.n)
        self._graphs: dict[tuple[int, int], torch.cuda.CUDAGraph] = {}
        torch.cuda.synchronize()

    def load(self, px=None, dx=None, kcache=None, vcache=None, block_table=None) -> None:
        """Overwrite workload inputs in place (captured decode graphs keep
        their pointers): prefill input [T, h], decode input [B, h], logical
        K/V caches [blocks, Hkv, page, d] (packed here into the device page
        layout) and the decode block table [B, pages]."""
        if px is not None:
            self.px.copy_(px)
        if dx is not None:
            self.dx.copy_(dx)
        if kcache is not None:
            self.dcache.k[: kcache.shape[0]].copy_(lib.kv_pack(kcache))
        if vcache is not None:
            self.dcache.v[: vcache.shape[0]].copy_(lib.kv_pack(vcache))
        if block_table is not None:
            self.block_table.copy_(block_table)
            pos, slots = decode_slots(self.block_table, self.ctx)
            self.d_pos.copy_(pos)
            self.d_slots.copy_(slots)
        torch.cuda.synchronize()

    # ------------------------------------------------------------- launches
    def prefill_layer(self, ps: PhaseStreams, timers=None, x=None, y=None, cta_trace=None) -> int:
        x = self.px if x is None else x
        y = self.py if y is None else y
        return self.layer.prefill(x, y, self.psc, self.p_cu, 1, self.T, self.p_pos, self.p_slots,
                                  self.pcache, ps.sms, ps.torch_stream, timers, cta_trace)

    def decode_layer(self, ds: PhaseStreams) -> int:
        return self.layer.decode(self.dx, self.dy, self.dsc, self.ctx, self.d_pos, self.d_slots,
                                 self.block_table, self.dcache, ds.sms, ds.torch_stream)

    def decode_graph(self, ds: PhaseStreams):
        """CUDA graph of one decode layer-step captured on the phase's stream."""
        key = (ds.stream, ds.sms)
        g = self._graphs.get(key)
        if g is None:
            with torch.cuda.stream(ds.torch_stream):
                self.decode_layer(ds)  # warm (tensor maps, attributes)
                ds.torch_stream.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=ds.torch_stream):
                    self.decode_layer(ds)
            torch.cuda.synchronize()
            self._graphs[key] = g
        return g

    def launches_per_decode_step(self, sms: int) -> int:
        """Kernels in one decode layer-step on `sms` SMs (the CUDA graph's nodes)."""
        m = self.model
        return 7 + lib.decode_attn_launches(self.B, m.num_heads, m.num_kv_heads, m.head_dim,
                                            self.block_table.shape[1], PAGE, sms)

    # --------------------------------------------------------------- timing
    def isolated(self, phase: int, sms: int, reps: int = 5) -> float:
        """Median seconds of one layer pass of `phase` alone on `sms` SMs."""
        st = self.pool.phase(phase, sms)
        times = []
        g = self.decode_graph(st) if phase == DECODE else None
        with torch.cuda.stream(st.torch_stream):
            for _ in range(reps + 1):
                lib.hold(st.torch_stream, 200_000)
                a, b = _ev(), _ev()
                a.record(st.torch_stream)
                if phase == PREFILL:
                    self.prefill_layer(st)
                else:
                    g.replay()
                b.record(st.torch_stream)
                times.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in times[1:])
        return ms[len(ms) // 2] * 1e-3

    def corun(self, pm: int, dm: int, steps: int, decode_per_step, time_upgate: bool = False,
              copy_in=None, copy_out=None, time_groups: bool = False, cta_trace=None) -> CoRunResult:
        """`steps` prefill layers on pm SMs co-executed with
        decode layer-steps on dm SMs (`decode_schedule`).  time_upgate:
        events around the mlp_up_gate GEMM only (the roofline kernel);
        time_groups: around every kernel group (diagnostic: the extra events
        between launches cost their programmatic-launch overlap)."""
        ps, ds = self.pool.split(pm, dm)
        g = self.decode_graph(ds)
        ctrl = torch.cuda.current_stream(self.dev)
        start, end_p, end_d = _ev(), _ev(), _ev()
        p_ev = [(_ev(), _ev()) for _ in range(steps)]
        timed = GROUPS if time_groups else (("mlp_up_gate",) if time_upgate else ())
        ug_ev = [{g: (_ev(), _ev()) for g in timed} for _ in range(steps)] if timed else None
        sched = decode_schedule(steps, decode_per_step)
        D = sum(sched)
        d_ev = [(_ev(), _ev()) for _ in range(D)]
        torch.cuda._sleep(400_000)
        start.record(ctrl)
        ps.torch_stream.wait_event(start)
        ds.torch_stream.wait_event(start)
        # interleave host enqueue so neither stream starves
        di = 0
        for s in range(steps):
            with torch.cuda.stream(ps.torch_stream):
                if copy_in is not None:
                    copy_in(PREFILL, ps.torch_stream)
                p_ev[s][0].record(ps.torch_stream)
                self.prefill_layer(ps, ug_ev[s] if ug_ev else None, cta_trace=cta_trace if s == steps - 1 else None)
                p_ev[s][1].record(ps.torch_stream)
                if copy_out is not None:
                    copy_out(PREFILL, ps.torch_stream)
            with torch.cuda.stream(ds.torch_stream):
                for _ in range(sched[s]):
                    if copy_in is not None:
                        copy_in(DECODE, ds.torch_stream)
                    d_ev[di][0].record(ds.torch_stream)
                    g.replay()
                    d_ev[di][1].record(ds.torch_stream)
                    if copy_out is not None:
                        copy_out(DECODE, ds.torch_stream)
                    di += 1
        end_p.record(ps.torch_stream)
        end_d.record(ds.torch_stream)
        torch.cuda.synchronize()
        span = max(start.elapsed_time(end_p), start.elapsed_time(end_d)) * 1e-3
        res = CoRunResult(pm, dm, steps, D, span, steps * self.T, D * self.B)
        res.prefill_layer_s = [a.elapsed_time(b) * 1e-3 for a, b in p_ev]
        res.decode_layer_s = [a.elapsed_time(b) * 1e-3 for a, b in d_ev]
        res.prefill_window_s = [(start.elapsed_time(a) * 1e-3, start.elapsed_time(b) * 1e-3) for a, b in p_ev]
        res.decode_window_s = [(start.elapsed_time(a) * 1e-3, start.elapsed_time(b) * 1e-3) for a, b in d_ev]
        if ug_ev:
            res.upgate_s = [a.elapsed_time(b) * 1e-3 for a, b in (e["mlp_up_gate"] for e in ug_ev)]
            res.group_s = {g: statistics.median(e[g][0].elapsed_time(e[g][1]) * 1e-3 for e in ug_ev)
                           for g in timed}
        return res

    def corun_e2e(self, pm: int, dm: int, steps: int, decode_per_step, host_px, host_py,
                  host_dx, host_dy) -> CoRunResult:
        """`corun` end to end from pinned host memory: every prefill layer's
        input is copied host->device and its output device->host, every
        decode step's input/output likewise.  Prefill copies run on their own
        copy-engine streams, double-buffered so step s+1's input lands and
        step s-1's output drains while step s computes (the serving
        pipeline); decode inputs / outputs (B x hidden per step) are read /
        written in place in pinned host memory by a copy kernel on the decode
        partition (UVA zero-copy), in-stream with the step."""
        ps, ds = self.pool.split(pm, dm)
        g = self.decode_graph(ds)
        sched = decode_schedule(steps, decode_per_step)
        ctrl = torch.cuda.current_stream(self.dev)
        h2d, d2h = torch.cuda.Stream(self.dev), torch.cuda.Stream(self.dev)
        xs = [self.px, torch.empty_like(self.px)]
        ys = [self.py, torch.empty_like(self.py)]
        in_ready = [_ev() for _ in range(steps)]
        done = [_ev() for _ in range(steps)]
        out_done = [_ev() for _ in range(steps)]
        start, end_p, end_d, end_o = _ev(), _ev(), _ev(), _ev()
        torch.cuda._sleep(400_000)
        start.record(ctrl)
        for st in (ps.torch_stream, ds.torch_stream, h2d, d2h):
            st.wait_event(start)

        chunks = max(1, getattr(self, "e2e_chunks", 4))  # prefill copies in 4 pieces
        pio = getattr(self, "e2e_prefill_io", True)
        dio = getattr(self, "e2e_decode_io", True)
        bounds = [self.T * i // chunks for i in range(chunks + 1)]

        def load(s):
            with torch.cuda.stream(h2d):
                if s >= 2:
                    h2d.wait_event(done[s - 2])  # buffer s%2 free once step s-2 computed
                if pio:
                    for a, b in zip(bounds, bounds[1:]):
                        xs[s % 2][a:b].copy_(host_px[a:b], non_blocking=True)
                in_ready[s].record(h2d)

        load(0)
        for s in range(steps):
            if s + 1 < steps:
                load(s + 1)
            with torch.cuda.stream(ps.torch_stream):
                ps.torch_stream.wait_event(in_ready[s])
                if s >= 2:
                    ps.torch_stream.wait_event(out_done[s - 2])  # ys[s%2] drained
                self.prefill_layer(ps, None, xs[s % 2], ys[s % 2])
                done[s].record(ps.torch_stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done[s])
                if pio:
                    for a, b in zip(bounds, bounds[1:]):
                        host_py[a:b].copy_(ys[s % 2][a:b], non_blocking=True)
                out_done[s].record(d2h)
            with torch.cuda.stream(ds.torch_stream):
                for _ in range(sched[s]):
                    # the step's B x hidden input / output cross PCIe through
                    # the decode partition's SMs (zero-copy, hp_copy_rows), so
                    # they never queue on a copy engine behind the prefill
                    # side's 34 MB transfers
                    if dio:
                        lib.copy_rows(host_dx, self.dx, ds.sms, ds.torch_stream)
                    g.replay()
                    if dio:
                        lib.copy_rows(self.dy, host_dy, ds.sms, ds.torch_stream)
        end_p.record(ps.torch_stream)
        end_d.record(ds.torch_stream)
        end_o.record(d2h)
        torch.cuda.synchronize()
        span = max(start.elapsed_time(e) for e in (end_p, end_d, end_o)) * 1e-3
        return CoRunResult(pm, dm, steps, sum(sched), span, steps * self.T, sum(sched) * self.B)

    def corun_hbm(self, pm: int, dm: int, steps: int = 2) -> dict:
        """North-star rooflines at ONE co-executed split: prefill layers on
        pm SMs (per-group CUDA events around the four GEMMs) while the dm-SM
        side streams back-to-back decode-attention launches (B sequences of
        context C) for the whole prefill window.  Returns the GEMMs' TFLOP/s
        and the attention's algorithmic GB/s over the launches that ran
        entirely inside the prefill window -- both measured at the same time
        on the device."""
        ps, ds = self.pool.split(pm, dm)
        m = self.model
        qkv = self.dsc.qkv[:self.B]

        def attn():
            lib.decode_attn(qkv, self.dcache.k, self.dcache.v, self.block_table, self.ctx, self.dsc.attn[:self.B],
                            m.num_heads, m.num_kv_heads, m.head_dim, PAGE, self.layer.scale, ws=self.dsc.attn_ws,
                            max_ctas=ds.sms, stream=ds.torch_stream)

        t_p = self.isolated(PREFILL, pm, reps=2)
        with torch.cuda.stream(ds.torch_stream):
            attn()  # warm
        a0, a1 = _ev(), _ev()
        with torch.cuda.stream(ds.torch_stream):
            lib.hold(ds.torch_stream, 200_000)
            a0.record(ds.torch_stream)
            for _ in range(20):
                attn()
            a1.record(ds.torch_stream)
        torch.cuda.synchronize()
        t_a = a0.elapsed_time(a1) * 1e-3 / 20
        n_attn = int(steps * t_p / t_a * 1.3) + 4
        ctrl = torch.cuda.current_stream(self.dev)
        start = _ev()
        p_ev = [(_ev(), _ev()) for _ in range(steps)]
        g_ev = [{g: (_ev(), _ev()) for g in GROUPS} for _ in range(steps)]
        d_ev = [(_ev(), _ev()) for _ in range(n_attn)]
        torch.cuda._sleep(400_000)
        start.record(ctrl)
        ps.torch_stream.wait_event(start)
        ds.torch_stream.wait_event(start)
        with torch.cuda.stream(ds.torch_stream):
            for e0, e1 in d_ev:
                e0.record(ds.torch_stream)
                attn()
                e1.record(ds.torch_stream)
        with torch.cuda.stream(ps.torch_stream):
            for s in range(steps):
                p_ev[s][0].record(ps.torch_stream)
                self.prefill_layer(ps, g_ev[s])
                p_ev[s][1].record(ps.torch_stream)
        torch.cuda.synchronize()
        win = [(start.elapsed_time(a) * 1e-3, start.elapsed_time(b) * 1e-3) for a, b in p_ev]
        p0, p1 = win[0][0], win[-1][1]
        inside = [b - a for a, b in ((start.elapsed_time(x) * 1e-3, start.elapsed_time(y) * 1e-3) for x, y in d_ev)
                  if a >= p0 and b <= p1]
        gemm_s = statistics.median(sum(e[g][0].elapsed_time(e[g][1]) * 1e-3 for g in GROUPS if g != "attn")
                                   for e in g_ev)
        h = m.hidden
        gemm_flops = 2.0 * self.T * h * (m.qkv_out_dim + h + 3 * mlp_width(m))
        return {"pm": pm, "dm": dm, "T": self.T, "prefill_layers": steps,
                "decode_attn_launches_inside": len(inside),
                "decode_attn_gbs": self.decode_attn_bytes() / statistics.median(inside) / 1e9 if inside else None,
                "decode_attn_alone_gbs": self.decode_attn_bytes() / t_a / 1e9,
                "prefill_gemm_tflops": gemm_flops / gemm_s / 1e12,
                "prefill_layer_us": 1e6 * statistics.median(b - a for a, b in win)}

    def measured_idle(self, pm: int, dm: int, decode_per_step) -> dict:
        """SM idle of the co-run MEASURED on the device (config 3's method
        inside config 2): the last of three co-run prefill layers records
        every CTA's {smid, start, end} (%globaltimer) for its five kernel
        groups while the decode graph replays on the dm side.  Per group:
        measured idle = 1 - sum(CTA busy) / (pm x group span), beside the
        wave model's wave_stats(units, 1, slots) (perf_model.py:157-169).
        Whole co-run (prefill layer window): 1 - (prefill CTA busy + dm x
        decode busy) / (N x window); the two RMSNorm launches and the
        decode kernels' intra-graph gaps count as busy only where timed."""
        from ..perf_model import wave_stats

        N, T, m = self.n, self.T, self.model
        traces = {g: torch.zeros(N, 3, dtype=torch.int64, device=self.dev) for g in GROUPS}
        r = self.corun(pm, dm, 3, decode_per_step, time_groups=True, cta_trace=traces)
        w = self.layer.W
        units = {}
        for g, wt in (("qkv", w.w_qkv), ("o_proj", w.w_o), ("mlp_up_gate", w.w_ug), ("mlp_down", w.w_down)):
            _, tiles, cpt = lib.gemm_plan(T, wt.shape[0], wt.shape[1], pm)
            units[g] = (tiles, pm // cpt)
        units["attn"] = (-(-T // 256) * m.num_heads, pm)
        groups, busy_sm_s = {}, 0.0
        for g in GROUPS:
            idle, span, ctas = lib.cta_idle(traces[g], pm)
            busy_sm_s += (1.0 - idle) * pm * span
            groups[g] = {"measured_idle": idle, "predicted_idle": wave_stats(units[g][0], 1, units[g][1]).idle_ratio,
                         "span_us": 1e6 * span, "ctas": ctas, "units": units[g][0], "slots": units[g][1]}
        p0, p1 = r.prefill_window_s[-1]
        dec = sum(max(0.0, min(p1, b) - max(p0, a)) for a, b in r.decode_window_s)
        window = p1 - p0
        tot_span = sum(v["span_us"] for v in groups.values())
        return {"groups": groups,
                "prefill_partition_measured": sum(v["measured_idle"] * v["span_us"] for v in groups.values()) / tot_span,
                "prefill_partition_predicted": sum(v["predicted_idle"] * v["span_us"] for v in groups.values()) / tot_span,
                "corun_measured": 1.0 - (busy_sm_s + dm * dec) / (N * window),
                "window_us": 1e6 * window, "decode_busy_in_window_us": 1e6 * dec}

    def time_sliced(self, steps: int, decode_per_step) -> CoRunResult:
        """Same work, one full-GPU stream: prefill layer then its decode steps."""
        st = self.pool.full(PREFILL)
        g = self.decode_graph(st)
        start, end = _ev(), _ev()
        p_ev = [(_ev(), _ev()) for _ in range(steps)]
        sched = decode_schedule(steps, decode_per_step)
        D = sum(sched)
        d_ev = [(_ev(), _ev()) for _ in range(D)]
        with torch.cuda.stream(st.torch_stream):
            torch.cuda._sleep(400_000)
            start.record(st.torch_stream)
            di = 0
            for s in range(steps):
                p_ev[s][0].record(st.torch_stream)
                self.prefill_layer(st)
                p_ev[s][1].record(st.torch_stream)
                for _ in range(sched[s]):
                    d_ev[di][0].record(st.torch_stream)
                    g.replay()
                    d_ev[di][1].record(st.torch_stream)
                    di += 1
            end.record(st.torch_stream)
        torch.cuda.synchronize()
        res = CoRunResult(self.n, self.n, steps, D, start.elapsed_time(end) * 1e-3, steps * self.T,
                          D * self.B)
        res.prefill_layer_s = [a.elapsed_time(b) * 1e-3 for a, b in p_ev]
        res.decode_layer_s = [a.elapsed_time(b) * 1e-3 for a, b in d_ev]
        res.prefill_window_s = [(start.elapsed_time(a) * 1e-3, start.elapsed_time(b) * 1e-3) for a, b in p_ev]
        res.decode_window_s = [(start.elapsed_time(a) * 1e-3, start.elapsed_time(b) * 1e-3) for a, b in d_ev]
        return res

    def chunked(self, chunk: int, reps: int = 1) -> dict:
        """The lockstep chunked-prefill baseline (reference _ChunkedSim,
        engine.py:741-800; SGLang-style hybrid batches) on real kernels, full
        GPU: every iteration carries the B decode tokens plus the next
        chunk - B tokens of the T-token prompt (prefix-aware attention over
        the chunks already cached).  Returns layer-level tokens/s, TTFT (all
        iterations until the prompt is done) and TPOT (median iteration)."""
        st = self.pool.full(PREFILL)
        take = max(1, chunk - self.B)
        plan = []
        p = 0
        while p < self.T:
            n = min(take, self.T - p)
            plan.append((n, p))
            p += n
        dev = self.dev
        i32 = dict(dtype=torch.int32, device=dev)
        args = []
        for n, p in plan:
            tot = n + self.B
            pos = torch.cat([torch.arange(p, p + n, **i32), self.d_pos])
            slots = torch.cat([self.chunk_pages[0, torch.arange(p, p + n, device=dev) // PAGE] * PAGE
                               + torch.arange(p, p + n, **i32) % PAGE, self.d_slots])
            args.append((tot, n, torch.tensor([0, n], **i32), torch.tensor([p], **i32), pos, slots))
        xb = torch.randn(max(a[0] for a in args), self.model.hidden, device=dev).to(torch.bfloat16)
        yb = torch.empty_like(xb)

        def run_iter(a):
            tot, n, cu, prior, pos, slots = a
            self.layer.hybrid(xb[:tot], yb[:tot], self.psc, self.dsc, n, cu, 1, n, prior, self.chunk_pages,
                              self.ctx, self.block_table, pos, slots, self.dcache, st.sms, st.torch_stream)

        with torch.cuda.stream(st.torch_stream):
            for a in args:  # warm (tensor maps)
                run_iter(a)
        torch.cuda.synchronize()
        evs = []
        with torch.cuda.stream(st.torch_stream):
            torch.cuda._sleep(400_000)
            for _ in range(reps):
                for a in args:
                    e0, e1 = _ev(), _ev()
                    e0.record(st.torch_stream)
                    run_iter(a)
                    e1.record(st.torch_stream)
                    evs.append((e0, e1))
        torch.cuda.synchronize()
        it = [a.elapsed_time(b) * 1e-3 for a, b in evs]
        per_prompt = sum(it) / reps
        tokens = (self.T + self.B * len(plan))
        return {"chunk": chunk, "iterations_per_prompt": len(plan), "tokens_per_s": tokens / per_prompt,
                "ttft_us": 1e6 * per_prompt, "tpot_p50_us": 1e6 * statistics.median(it)}

    def decode_attn_bytes(self) -> int:
        """Algorithmic HBM bytes of one decode-attention launch (workload.py:
        184-188): K+V over every context, the new token's K/V, q and out."""
        m = self.model
        kv_dim = m.num_kv_heads * m.head_dim
        return self.B * (self.C * 2 * kv_dim * 2 + 2 * kv_dim * 2 + 2 * m.hidden * 2)

    def sm_ingest_gbs(self, sms: int, reps: int = 3) -> float:
        """Raw HBM -> SM ingest of an `sms`-SM partition: the bulk-copy probe
        (hp_membw method 1, TMA 1-D copies into a 6 x 32 KB shared-memory
        ring, nothing read back) over a 1 GiB buffer, GB/s, median of `reps`.
        The per-SM ceiling any reader that stages through shared memory works
        under; one that also reads every byte back (ld.shared, 8 reader
        warps) keeps ~80 % of it (hp_membw_stage, profiles/r02_decode_ingest.md)."""
        st = self.pool.phase(DECODE, sms)
        buf = torch.empty(1 << 30, dtype=torch.uint8, device=self.dev)
        out = torch.zeros(4, device=self.dev)
        evs = []
        with torch.cuda.stream(st.torch_stream):
            lib.membw(buf, st.sms, 1, out, stream=st.torch_stream)
            for _ in range(reps):
                lib.hold(st.torch_stream, 100_000)
                a, b = _ev(), _ev()
                a.record(st.torch_stream)
                lib.membw(buf, st.sms, 1, out, stream=st.torch_stream)
                b.record(st.torch_stream)
                evs.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(a.elapsed_time(b) for a, b in evs) * 1e-3
        del buf
        return (1 << 30) / t / 1e9

    def decode_attn_gbs(self, sms: int, reps: int = 10) -> float:
        """Decode attention alone on `sms` SMs, GB/s algorithmic: `reps`
        back-to-back launches per event pair, median of three pairs."""
        st = self.pool.phase(DECODE, sms)
        m = self.model
        qkv = self.dsc.qkv[:self.B]
        def launch():
            lib.decode_attn(qkv, self.dcache.k, self.dcache.v, self.block_table, self.ctx,
                            self.dsc.attn[:self.B], m.num_heads, m.num_kv_heads, m.head_dim, PAGE,
                            self.layer.scale, ws=self.dsc.attn_ws, max_ctas=st.sms, stream=st.torch_stream)

        # back-to-back launches between two events: the steady-state
        # per-launch time (each launch streams 269 MB > L2, so no reuse)
        evs = []
        with torch.cuda.stream(st.torch_stream):
            launch()
            for _ in range(3):
                lib.hold(st.torch_stream, 200_000)
                a, b = _ev(), _ev()
                a.record(st.torch_stream)
                for _ in range(reps):
                    launch()
                b.record(st.torch_stream)
                evs.append((a, b))
        torch.cuda.synchronize()
        t = statistics.median(a.elapsed_time(b) for a, b in evs) * 1e-3 / reps
        return self.decode_attn_bytes() / t / 1e9

    # ------------------------------------------------------------ workload
    def prefill_flops(self) -> float:
        m = self.model
        h = m.hidden
        gemm = 2.0 * self.T * h * (m.qkv_out_dim + h + 3 * mlp_width(m))
        attn = 2.0 * self.T * self.T * h  # causal: 4 T^2 h / 2
        return gemm + attn

    def upgate_flops(self) -> float:
        return 4.0 * self.T * mlp_width(self.model) * self.model.hidden
