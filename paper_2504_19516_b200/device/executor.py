"""B200Executor: the reference's device seam, executed on hardware.

Implements the `GroundTruthOracle` protocol (reference engine.py:159-208):

  prefill_layer_s(es)   one prefill layer over es.prefill_lens on
                        es.prefill_sms SMs, with the decode side of `es`
                        running concurrently on es.decode_sms SMs
  decode_step_s(es)     one decode step (all model layers) for
                        es.decode_ctx_lens on es.decode_sms SMs, with the
                        prefill side of `es` running concurrently
  hybrid_iteration_s(chunks, decode_ctx_lens, sms)
                        one lockstep hybrid batch (chunked-prefill baseline)
  alpha(phase, sms, tokens)        measured / SRM at a canonical shape
  contention_bw(sms, prefill_len)  HBM bandwidth of `sms` SMs next to a
                                   prefill on the remaining SMs

so `engine.run(cfg, trace, oracle=B200Executor(...))` drives the
reference's event loop with CUDA-event measurements of the real kernels
confined to green-context partitions (PartitionPool) instead of the
synthetic surfaces.  Decisions, queueing and reports stay the reference's.

By default every layer of a decode step has identical cost, so a step is
measured as one decode layer (queued ahead of the timer, so host launch
latency is excluded) times `model.num_layers`, and a prefill layer as one
resident layer.  With `full_model=True` every layer is resident (distinct
random weights, per-layer KV pools): a decode step is measured over all
layers and a prefill step over `l_step` distinct layers.  K/V for arbitrary
decode batches come from a page pool addressed modulo its size (the bytes
streamed are what the timing depends on).
"""

from __future__ import annotations

import math

import torch

from ..errors import InvalidArgumentError
from ..perf_model import ExecutionState, GpuSpec, srm_decode_step_s, srm_prefill_layer_s
from ..workload import ModelSpec
from . import lib
from .layer import PAGE, DecodeScratch, DeviceLayer, KVCache, LayerWeights, PrefillScratch, decode_slots
from .partition import DECODE, PREFILL, PartitionPool


def _ev():
    return torch.cuda.Event(enable_timing=True)


class B200Executor:
    def __init__(self, model: ModelSpec, gpu: GpuSpec, device: int = 0, seed: int = 0,
                 max_prefill_tokens: int = 32768, max_decode_batch: int = 256,
                 pool_tokens: int = 1 << 21, sm_step: int = 8, pool: PartitionPool | None = None,
                 memo: bool = False, full_model: bool = False, l_step: int = 4):
        """full_model=True keeps every layer of `model` resident (distinct
        random weights, per-layer paged KV pools): a decode step is measured
        as the whole model's layers back to back and a prefill step as
        `l_step` distinct layers (scheduler.py:47 l_step), instead of one
        resident layer scaled by the layer count."""
        if model.head_dim not in (64, 128):
            raise InvalidArgumentError("B200Executor supports head_dim 64 or 128")
        self.model = model
        self.gpu = gpu
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        self.pool = pool or PartitionPool(device, granularity=max(8, sm_step))
        if gpu.num_sms != self.pool.n:
            raise InvalidArgumentError(
                f"GpuSpec has {gpu.num_sms} SMs but the device has {self.pool.n}; "
                "use perf_model.b200_spec() (or [gpu] num_sms = 148)")
        gen = torch.Generator(device="cpu")
        gen.manual_seed(seed)
        self.full_model = full_model
        self.l_step = max(1, min(l_step, model.num_layers)) if full_model else 1
        max_pos = max(max_prefill_tokens, 1 << 15) + 1
        if full_model:
            g = torch.Generator(device=self.dev)
            g.manual_seed(seed)
            self.layers = [DeviceLayer(model, LayerWeights.random_device(model, self.dev, g), self.dev,
                                       max_pos=max_pos) for _ in range(model.num_layers)]
            for lyr in self.layers[1:]:
                lyr.rope = self.layers[0].rope
        else:
            self.layers = [DeviceLayer(model, LayerWeights.random(model, self.dev, gen), self.dev,
                                       max_pos=max_pos)]
        self.layer = self.layers[0]
        h = model.hidden
        bf = dict(dtype=torch.bfloat16, device=self.dev)
        self.max_prefill_tokens = max_prefill_tokens
        self.px = torch.randn(max_prefill_tokens, h, generator=gen).to(**bf)
        self.py = torch.empty_like(self.px)
        self.psc = PrefillScratch(model, max_prefill_tokens, self.dev)
        self.pcaches = [KVCache(-(-max_prefill_tokens // PAGE), model.num_kv_heads, model.head_dim, self.dev)
                        for _ in range(self.l_step)]
        self.pcache = self.pcaches[0]
        self.pool_blocks = max(1, pool_tokens // PAGE)
        self.dcaches = [KVCache(self.pool_blocks, model.num_kv_heads, model.head_dim, self.dev)
                        for _ in range(len(self.layers))]
        self.dcache = self.dcaches[0]
        self.max_decode_batch = max_decode_batch
        self.dx = torch.randn(max_decode_batch, h, generator=gen).to(**bf)
        self.dy = torch.empty_like(self.dx)
        self.dsc = DecodeScratch(model, max_decode_batch, 1024, self.dev, max_ctas=self.pool.n)
        self.max_ctx = 1024 * PAGE  # contexts the decode scratch's block tables address
        self.calls = {"prefill": 0, "decode": 0}
        self._warm: set = set()
        # memo=True: reuse a measurement for states with the same partition,
        # prefill lengths, decode batch size and mean KV pages per sequence
        # (the quantities the step time depends on) -- bounds the GPU time of
        # long serving traces; off by default (every call measures)
        self.memo = {} if memo else None
        self.memo_hits = 0

    # ------------------------------------------------------------ workloads
    def _prefill_args(self, lens):
        lens = [int(x) for x in lens]
        T = sum(lens)
        if T > self.max_prefill_tokens:
            raise InvalidArgumentError(f"prefill of {T} tokens exceeds max_prefill_tokens")
        cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0).tolist()), dtype=torch.int32, device=self.dev)
        pos = torch.cat([torch.arange(L, dtype=torch.int32) for L in lens]).to(self.dev)
        slots = torch.arange(T, dtype=torch.int32, device=self.dev)
        return T, cu, len(lens), max(lens), pos, slots

    def _decode_args(self, ctx_lens):
        B = len(ctx_lens)
        if B > self.max_decode_batch:
            raise InvalidArgumentError(f"decode batch {B} exceeds max_decode_batch")
        pages = [-(-int(c) // PAGE) for c in ctx_lens]
        mp = max(pages)
        bt = torch.zeros(B, mp, dtype=torch.int64)
        nxt = 0
        for i, p in enumerate(pages):
            bt[i, :p] = (torch.arange(p) + nxt) % self.pool_blocks
            nxt += p
        bt = bt.to(torch.int32).to(self.dev)
        ctx = torch.tensor([int(c) for c in ctx_lens], dtype=torch.int32, device=self.dev)
        pos, slots = decode_slots(bt, ctx)
        return B, ctx, bt, pos, slots

    def _launch_prefill(self, ps, args):
        """One prefill unit: l_step distinct layers (1 unless full_model)."""
        T, cu, nseq, mx, pos, slots = args
        x, y = self.px[:T], self.py[:T]
        for i in range(self.l_step):
            self.layers[i].prefill(x, y, self.psc, cu, nseq, mx, pos, slots, self.pcaches[i], ps.sms,
                                   ps.torch_stream)
            x, y = y, x

    def _launch_decode(self, ds, args):
        """One decode unit: every resident layer (the whole model if full_model)."""
        B, ctx, bt, pos, slots = args
        x, y = self.dx[:B], self.dy[:B]
        for lyr, cache in zip(self.layers, self.dcaches):
            lyr.decode(x, y, self.dsc, ctx, pos, slots, bt, cache, ds.sms, ds.torch_stream)
            x, y = y, x

    # --------------------------------------------------------------- timing
    def _measure(self, phase: str, es: ExecutionState) -> float:
        """Seconds of one layer of `phase` under the co-execution state `es`."""
        n = self.pool.n
        pm = es.prefill_sms if es.prefill_lens else 0
        dm = es.decode_sms if es.decode_ctx_lens else 0
        ps, ds = self.pool.split(pm, dm)
        pargs = self._prefill_args(es.prefill_lens) if ps is not None else None
        dargs = self._decode_args(es.decode_ctx_lens) if ds is not None else None
        main, other = (ps, ds) if phase == "prefill" else (ds, ps)
        run_main = self._launch_prefill if phase == "prefill" else self._launch_decode
        run_other = self._launch_decode if phase == "prefill" else self._launch_prefill
        margs, oargs = (pargs, dargs) if phase == "prefill" else (dargs, pargs)
        if main is None:
            raise InvalidArgumentError(f"{phase} phase has no SMs in {es}")
        cover = self._cover_count(phase, es) if other is not None else 0
        key = (phase, pm, dm, es.prefill_lens, es.decode_ctx_lens)
        if key not in self._warm:  # first launch of a shape: tensor maps, module load
            with torch.cuda.stream(main.torch_stream):
                run_main(main, margs)
            if other is not None:
                with torch.cuda.stream(other.torch_stream):
                    run_other(other, oargs)
            torch.cuda.synchronize(self.dev)
            self._warm.add(key)
        ctrl = torch.cuda.current_stream(self.dev)
        start = _ev()
        a, b = _ev(), _ev()
        # hold the GPU while the host queues everything (~10 launches per
        # layer, tens of us each through ctypes), so host latency stays out
        torch.cuda._sleep(400_000 + 300_000 * (1 + cover))
        start.record(ctrl)
        main.torch_stream.wait_event(start)
        if other is not None:
            other.torch_stream.wait_event(start)
            # keep the other phase busy for the whole measured layer
            with torch.cuda.stream(other.torch_stream):
                for _ in range(cover):
                    run_other(other, oargs)
        with torch.cuda.stream(main.torch_stream):
            a.record(main.torch_stream)
            run_main(main, margs)
            b.record(main.torch_stream)
        torch.cuda.synchronize(self.dev)
        self.calls[phase] += 1
        return a.elapsed_time(b) * 1e-3

    def _cover_count(self, phase: str, es: ExecutionState) -> int:
        """How many layers of the other phase overlap one layer of `phase`."""
        # SRM estimates of one launch unit of each phase (l_step prefill
        # layers; one decode layer, or the whole step with full_model)
        p = (self.l_step * srm_prefill_layer_s(es, self.model, self.gpu)
             if es.prefill_lens and es.prefill_sms else 0.0)
        d = (srm_decode_step_s(es, self.model, self.gpu) * len(self.layers) / self.model.num_layers
             if es.decode_ctx_lens and es.decode_sms else 0.0)
        if phase == "prefill":
            return max(1, min(64, math.ceil(3.0 * p / max(d, 1e-9))))
        return max(1, min(8, math.ceil(3.0 * d / max(p, 1e-9))))

    # -------------------------------------------------------- oracle protocol
    def _memo_key(self, phase: str, es: ExecutionState):
        ctx = es.decode_ctx_lens
        pages = -(-sum(int(c) for c in ctx) // PAGE) if ctx else 0
        return (phase, es.prefill_sms if es.prefill_lens else 0, es.decode_sms if ctx else 0,
                tuple(es.prefill_lens), len(ctx), round(pages / max(1, len(ctx))))

    def _measured(self, phase: str, es: ExecutionState) -> float:
        if self.memo is None:
            return self._measure(phase, es)
        key = self._memo_key(phase, es)
        v = self.memo.get(key)
        if v is None:
            v = self.memo[key] = self._measure(phase, es)
        else:
            self.memo_hits += 1
        return v

    def prefill_layer_s(self, es: ExecutionState) -> float:
        return self._measured("prefill", es) / self.l_step

    def decode_step_s(self, es: ExecutionState) -> float:
        return self.model.num_layers / len(self.layers) * self._measured("decode", es)

    def _hybrid_args(self, chunks, decode_ctx_lens):
        """Device inputs of one hybrid batch: chunk rows first, then decode
        rows; every sequence gets its own run of pool pages (mod pool size)."""
        chunks = [(int(n), int(p)) for n, p in chunks]
        ctxs = [int(c) for c in decode_ctx_lens]
        Tc = sum(n for n, _ in chunks)
        B = len(ctxs)
        T = Tc + B
        if T < 1:
            raise InvalidArgumentError("hybrid batch is empty")
        if T > self.max_prefill_tokens:
            raise InvalidArgumentError(f"hybrid batch of {T} tokens exceeds max_prefill_tokens")
        if B > self.max_decode_batch:
            raise InvalidArgumentError(f"decode batch {B} exceeds max_decode_batch")
        seqs = chunks + [(1, c - 1) for c in ctxs]
        pages = [-(-(n + p) // PAGE) for n, p in seqs]
        mp = max(pages)
        bt = torch.zeros(len(seqs), mp, dtype=torch.int64)
        pos, slots = [], []
        nxt = 0
        for i, ((n, p), pg) in enumerate(zip(seqs, pages)):
            bt[i, :pg] = (torch.arange(pg) + nxt) % self.pool_blocks
            nxt += pg
            ps = torch.arange(p, p + n)
            pos.append(ps)
            slots.append(bt[i, ps // PAGE] * PAGE + ps % PAGE)
        nc = len(chunks)
        d = dict(device=self.dev, dtype=torch.int32)
        offs = [0]
        for n, _ in chunks:
            offs.append(offs[-1] + n)
        cu = torch.tensor(offs, **d)
        return dict(T=T, Tc=Tc, cu=cu, max_chunk=max([n for n, _ in chunks] or [1]),
                    prior=torch.tensor([p for _, p in chunks] or [0], **d),
                    cbt=bt[:max(nc, 1)].to(**d), dctx=torch.tensor(ctxs or [1], **d),
                    dbt=bt[nc:].to(**d) if B else bt[:1].to(**d),
                    pos=torch.cat(pos).to(**d), slots=torch.cat(slots).to(**d))

    def _launch_hybrid(self, st, a):
        T = a["T"]
        x, y = self.px[:T], self.py[:T]
        for lyr, cache in zip(self.layers, self.dcaches):
            lyr.hybrid(x, y, self.psc, self.dsc, a["Tc"], a["cu"], a["cu"].shape[0] - 1, a["max_chunk"],
                       a["prior"], a["cbt"], a["dctx"], a["dbt"], a["pos"], a["slots"], cache, st.sms,
                       st.torch_stream)
            x, y = y, x

    def hybrid_iteration_s(self, chunks, decode_ctx_lens, sms: int) -> float:
        """One lockstep hybrid iteration (all layers) on `sms` SMs -- the
        chunked-prefill baseline's device call (reference engine.py:200-208,
        issued by _ChunkedSim._start_iteration engine.py:795-797).  Measured
        as one hybrid layer (prefix-aware paged prefill attention for the
        chunks, paged decode attention for the decode rows, GEMMs over the
        concatenated stream) times `model.num_layers`."""
        a = self._hybrid_args(chunks, decode_ctx_lens)
        st = self.pool.phase(PREFILL, sms)
        key = ("hybrid", sms, tuple(chunks), tuple(decode_ctx_lens))
        if key not in self._warm:
            with torch.cuda.stream(st.torch_stream):
                self._launch_hybrid(st, a)
            torch.cuda.synchronize(self.dev)
            self._warm.add(key)
        a_ev, b_ev = _ev(), _ev()
        with torch.cuda.stream(st.torch_stream):
            torch.cuda._sleep(400_000)
            a_ev.record(st.torch_stream)
            self._launch_hybrid(st, a)
            b_ev.record(st.torch_stream)
        torch.cuda.synchronize(self.dev)
        self.calls["hybrid"] = self.calls.get("hybrid", 0) + 1
        return self.model.num_layers / len(self.layers) * a_ev.elapsed_time(b_ev) * 1e-3

    def alpha(self, phase: str, sms: int, tokens: int) -> float:
        """Measured / SRM at a canonical shape of `tokens` on `sms` SMs."""
        if phase == "prefill":
            T = max(1, min(int(tokens), self.max_prefill_tokens))
            es = ExecutionState(prefill_lens=(T,), prefill_sms=sms)
            return self.prefill_layer_s(es) / srm_prefill_layer_s(es, self.model, self.gpu)
        from ..engine import canonical_decode_es

        # the reference's canonical batch (<= 256 sequences of ~1k, longer
        # contexts beyond 256k tokens) measured at its real token count; a
        # batch beyond the resident scratch keeps the token count with
        # max_decode_batch longer sequences
        es = canonical_decode_es(int(tokens), sms)
        if es.decode_batch > self.max_decode_batch or max(es.decode_ctx_lens) > self.max_ctx:
            # alpha is a ratio: beyond the resident scratch (max_decode_batch
            # sequences of <= max_ctx) it is measured at the largest batch
            bs = self.max_decode_batch
            tok = min(int(tokens), bs * self.max_ctx)
            ctx = max(1, tok // bs)
            es = ExecutionState(decode_ctx_lens=(ctx,) * (bs - 1) + (max(1, tok - ctx * (bs - 1)),),
                                decode_sms=sms)
        return self.decode_step_s(es) / srm_decode_step_s(es, self.model, self.gpu)

    def contention_bw(self, sms: int, co_prefill_len: int, nbytes: int = 1 << 30) -> float:
        """HBM bytes/s a stream on `sms` SMs attains while a prefill layer of
        `co_prefill_len` tokens runs on the other N - sms SMs."""
        buf = getattr(self, "_bwbuf", None)
        if buf is None or buf.numel() * 4 != nbytes:
            buf = self._bwbuf = torch.ones(nbytes // 4, dtype=torch.float32, device=self.dev)
            self._bwout = torch.zeros(4, device=self.dev)
        n = self.pool.n
        T = max(0, min(int(co_prefill_len), self.max_prefill_tokens))
        if T > 0 and sms < n:
            ps, ds = self.pool.split(n - sms, sms)
        else:
            ds, ps = self.pool.phase(DECODE, sms), None
        ctrl = torch.cuda.current_stream(self.dev)
        if not getattr(self, "_bw_warm", False):
            # first launch of the probe pays module loading / first-use costs
            with torch.cuda.stream(ds.torch_stream):
                lib.membw(buf, ds.sms, 1, self._bwout, stream=ds.torch_stream)
            torch.cuda.synchronize(self.dev)
            self._bw_warm = True
        start, a, b = _ev(), _ev(), _ev()
        torch.cuda._sleep(300_000)
        start.record(ctrl)
        if ps is not None:
            ps.torch_stream.wait_event(start)
            args = self._prefill_args([T])
            with torch.cuda.stream(ps.torch_stream):
                for _ in range(3):
                    self._launch_prefill(ps, args)
        ds.torch_stream.wait_event(start)
        with torch.cuda.stream(ds.torch_stream):
            a.record(ds.torch_stream)
            lib.membw(buf, ds.sms, 1, self._bwout, stream=ds.torch_stream)
            b.record(ds.torch_stream)
        torch.cuda.synchronize(self.dev)
        return nbytes / (a.elapsed_time(b) * 1e-3)
