"""Real-time co-executed serving: the reference's event loop on a wall clock,
driving a whole model on the B200 and generating real tokens.

The reference (`_ConcurrentSim`, engine.py:513-712) advances a heap by
`t + step_s` returned from its oracle (engine.py:599, 682).  `RealtimeSim`
keeps every decision the reference makes -- Algorithm 1 via
`schedule_prefill` / `set_balanced_sm` / `transition_handoff`, FCFS decode
via `schedule_decode`, KV admission, partition requests, `update_online`,
the TPOT window -- and replaces the oracle + heap with the device:

  * `_launch_prefill` enqueues `l_step` real prefill layers of the in-flight
    batch (packed prompts, paged KV writes) on the prefill partition's
    green-context stream and returns at once;
  * `_maybe_launch_decode` replays the WHOLE-MODEL decode step (embedding,
    all layers, final norm, LM head, greedy argmax) as ONE CUDA graph per
    batch bucket, captured on the decode partition's stream;
  * the loop polls the two phases' completion events; the completion times
    (CUDA events on the device timeline, aligned with the host clock at
    start) become the token timestamps, the measured step times feed
    `update_online` and `tpot_window` exactly where the reference feeds its
    oracle's numbers (engine.py:578, 673-675);
  * arrivals are released when the host clock reaches `arrival_s`, so the
    Python control plane's own cost lands on the timeline.

Tokens are real: every request is prefilled and greedily decoded through
the hp_* kernels; `generated[rid]` holds its token ids (tests compare them
with the CPU oracle for the tiny model).  With `trace_decisions=True` every
scheduling call logs the exact `SystemState` it saw, a snapshot of the
calibration store and the decision taken (tests re-run the reference's
scheduler on them and require identical decisions).
"""

from __future__ import annotations

import heapq
import time
from dataclasses import dataclass

import numpy as np
import torch

from .. import engine as E
from ..errors import InvalidArgumentError
from ..perf_model import ExecutionState
from ..scheduler import schedule_decode
from ..workload import ModelSpec, kv_bytes
from . import lib
from .layer import (EPS, PAGE, DecodeScratch, DeviceLayer, KVCache, LayerWeights, PrefillScratch,
                    decode_slots)
from .partition import PartitionPool

__all__ = ["ServingModel", "RealtimeSim", "RealtimeChunked", "kv_pages_for", "state_to_json", "state_from_json",
           "store_from_json"]

BUCKETS = (8, 16, 32, 64, 128, 256)


def _ev():
    return torch.cuda.Event(enable_timing=True)


def _idle(until_arrival, device_busy: bool) -> None:
    """Wait in the event loop: spin (event polls cost ~2 us) while a device
    step is in flight -- a sleep's ~60 us wake-up latency would sit on the
    GPU timeline between steps -- else sleep toward the next arrival."""
    if device_busy:
        return
    if until_arrival is not None and until_arrival > 2e-4:
        time.sleep(min(until_arrival - 1e-4, 1e-3))


def bucket_of(b: int) -> int:
    for k in BUCKETS:
        if b <= k:
            return k
    raise InvalidArgumentError(f"decode batch {b} exceeds the largest bucket {BUCKETS[-1]}")


class ServingModel:
    """A whole decoder resident in HBM for serving: L layers with paged KV
    pools of `kv_pages` pages each (page 0 is a scratch page that padded
    decode rows write to), embedding, final norm, LM head; separate scratch
    for the prefill and decode phases so both can run at once."""

    def __init__(self, model: ModelSpec, vocab: int, device, kv_pages: int, max_prefill_tokens: int,
                 max_pages_per_seq: int, max_batch: int = 256, seed: int = 0, weights=None, embed=None,
                 final_norm=None, lm_head=None, sms: int = 148):
        max_pages_per_seq = -(-max_pages_per_seq // 4) * 4  # 16-byte block-table rows (hp_copy_rows)
        self.model = model
        self.vocab = vocab
        self.dev = torch.device(device)
        self.kv_pages = kv_pages
        self.max_pages = max_pages_per_seq
        self.max_prefill_tokens = max_prefill_tokens
        self.max_batch = max_batch
        h, L = model.hidden, model.num_layers
        bf = dict(dtype=torch.bfloat16, device=self.dev)
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        if weights is None:
            weights = [LayerWeights.random_device(model, self.dev, g) for _ in range(L)]
        self.layers = [DeviceLayer(model, w, self.dev, max_pos=max_pages_per_seq * PAGE + 1) for w in weights]
        for lyr in self.layers[1:]:
            lyr.rope = self.layers[0].rope
        self.embed = embed if embed is not None else torch.randn(vocab, h, generator=g, device=self.dev).to(**bf)
        self.final_norm = final_norm if final_norm is not None else torch.ones(h, **bf)
        if lm_head is None:
            lm_head = (torch.randn(vocab, h, generator=g, device=self.dev) * 0.05).to(**bf)
        self.lm_head = lib.tile_weight(lm_head)
        self.caches = [KVCache(kv_pages, model.num_kv_heads, model.head_dim, self.dev) for _ in range(L)]
        # prefill phase
        self.psc = PrefillScratch(model, max_prefill_tokens, self.dev)
        self.pbuf = [torch.empty(max_prefill_tokens, h, **bf) for _ in range(2)]
        self.p_norm = torch.empty(max_batch, h, **bf)
        self.p_logits = torch.empty(max_batch, vocab, **bf)
        self.p_next = torch.zeros(max_batch, dtype=torch.int32, device=self.dev)
        self.h_p_next = torch.zeros(max_batch, dtype=torch.int32, pin_memory=True)
        # decode phase: static graph inputs / outputs
        self.dsc = DecodeScratch(model, max_batch, max_pages_per_seq, self.dev, max_ctas=sms)
        self.dbuf = [torch.empty(max_batch, h, **bf) for _ in range(2)]
        self.d_norm = torch.empty(max_batch, h, **bf)
        self.d_logits = torch.empty(max_batch, vocab, **bf)
        self.d_tok = torch.zeros(max_batch, dtype=torch.int32, device=self.dev)
        self.d_ctx = torch.ones(max_batch, dtype=torch.int32, device=self.dev)
        self.d_bt = torch.zeros(max_batch, max_pages_per_seq, dtype=torch.int32, device=self.dev)
        self.d_next = torch.zeros(max_batch, dtype=torch.int32, device=self.dev)
        self.h_in = torch.zeros(max_batch * (2 + max_pages_per_seq), dtype=torch.int32, pin_memory=True)
        self.h_d_next = torch.zeros(max_batch, dtype=torch.int32, pin_memory=True)
        nb = max(lib.gemm_swap_ws_bytes(max_batch, vocab, h, c) for c in range(1, 149))
        self.lm_ws = [torch.empty(nb // 4 + 1, dtype=torch.float32, device=self.dev) for _ in range(2)]
        self.lm_cnt = [torch.zeros(-(-vocab // 128) * 8, dtype=torch.int32, device=self.dev) for _ in range(2)]
        self._graphs: dict = {}
        self._gpool = torch.cuda.graph_pool_handle()  # one pool: decode steps never overlap
        torch.cuda.synchronize(self.dev)

    # ----------------------------------------------------------- prefill
    def prefill_layers(self, l0: int, l1: int, meta: dict, sms: int, stream) -> None:
        """Layers [l0, l1) over the packed prompts of `meta`; at l0 == 0 the
        input is the prompts' embedding, at l1 == L the last token of each
        prompt goes through the final norm + LM head + argmax and its id is
        copied to pinned host memory (h_p_next)."""
        T, nseq = meta["T"], meta["nseq"]
        with torch.cuda.stream(stream):
            if l0 == 0:
                torch.index_select(self.embed, 0, meta["tokens"], out=self.pbuf[0][:T])
            for li in range(l0, l1):
                x, y = self.pbuf[li % 2][:T], self.pbuf[(li + 1) % 2][:T]
                self.layers[li].prefill(x, y, self.psc, meta["cu"], nseq, meta["max_len"], meta["pos"],
                                        meta["slots"], self.caches[li], sms, stream)
            if l1 == self.model.num_layers:
                hid = self.pbuf[l1 % 2]
                last = self.p_norm[:nseq]
                torch.index_select(hid, 0, meta["last"], out=last)
                lib.rmsnorm(last, self.final_norm, last, EPS, sms, stream)
                self._lm_head(last, self.p_logits[:nseq], 0, sms, stream)
                self.p_next[:nseq].copy_(torch.argmax(self.p_logits[:nseq], dim=-1))
                lib.copy_rows(self.p_next.view(1, -1), self.h_p_next.view(1, -1), sms, stream)

    def hybrid_step(self, meta: dict, sms: int, stream) -> None:
        """One lockstep hybrid iteration through every layer (the chunked
        baseline, reference _ChunkedSim engine.py:741-800): prompt-chunk rows
        (cached prefixes via paged prefill attention) then one row per
        decoding request; the rows in meta["emit"] go through the LM head and
        their argmax ids land in h_p_next."""
        T, ne = meta["T"], meta["n_emit"]
        with torch.cuda.stream(stream):
            torch.index_select(self.embed, 0, meta["tokens"], out=self.pbuf[0][:T])
            for li, (lyr, cache) in enumerate(zip(self.layers, self.caches)):
                x, y = self.pbuf[li % 2][:T], self.pbuf[(li + 1) % 2][:T]
                lyr.hybrid(x, y, self.psc, self.dsc, meta["Tc"], meta["cu"], meta["n_chunks"], meta["max_chunk"],
                           meta["prior"], meta["cbt"], meta["dctx"], meta["dbt"], meta["pos"], meta["slots"],
                           cache, sms, stream)
            if ne:
                hid = self.pbuf[self.model.num_layers % 2]
                last = self.p_norm[:ne]
                torch.index_select(hid, 0, meta["emit"], out=last)
                lib.rmsnorm(last, self.final_norm, last, EPS, sms, stream)
                self._lm_head(last, self.p_logits[:ne], 0, sms, stream)
                self.p_next[:ne].copy_(torch.argmax(self.p_logits[:ne], dim=-1))
                lib.copy_rows(self.p_next.view(1, -1), self.h_p_next.view(1, -1), sms, stream)

    def _lm_head(self, x, out, which: int, sms: int, stream) -> None:
        if x.shape[0] <= 256:
            lib.gemm_swap(x, self.lm_head, out, self.lm_ws[which], self.lm_cnt[which], lib.EPI_STORE,
                          max_ctas=sms, stream=stream)
        else:
            lib.gemm(x, self.lm_head, out, lib.EPI_STORE, max_ctas=sms, stream=stream)

    # ------------------------------------------------------------ decode
    def _decode_body(self, b: int, sms: int, stream) -> None:
        tok, ctx, bt = self.d_tok[:b], self.d_ctx[:b], self.d_bt[:b]
        x = self.dbuf[0][:b]
        torch.index_select(self.embed, 0, tok, out=x)
        pos, slots = decode_slots(bt, ctx)
        for i, (lyr, cache) in enumerate(zip(self.layers, self.caches)):
            y = self.dbuf[(i + 1) % 2][:b]
            lyr.decode(x, y, self.dsc, ctx, pos, slots, bt, cache, sms, stream)
            x = y
        lib.rmsnorm(x, self.final_norm, self.d_norm[:b], EPS, sms, stream)
        self._lm_head(self.d_norm[:b], self.d_logits[:b], 1, sms, stream)
        self.d_next[:b].copy_(torch.argmax(self.d_logits[:b], dim=-1))

    def decode_graph(self, b: int, ps) -> torch.cuda.CUDAGraph:
        """The whole-model decode step for a batch bucket of `b` rows as one
        CUDA graph, captured on (and replayed into) the decode partition's
        stream `ps` (one graph per bucket and partition)."""
        key = (b, ps.stream, ps.sms)
        g = self._graphs.get(key)
        if g is None:
            st = ps.torch_stream
            with torch.cuda.stream(st):
                self._decode_body(b, ps.sms, st)  # warm (tensor maps, attributes)
                st.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st, pool=self._gpool):
                    self._decode_body(b, ps.sms, st)
            torch.cuda.synchronize(self.dev)
            self._graphs[key] = g
        return g

    def warm(self, pool: PartitionPool, buckets=BUCKETS, shares=None) -> int:
        """Capture every decode graph a run can replay -- each bucket on every
        decode share of the 8-SM grid plus the full device -- before the
        clock starts (a first-use capture costs tens of ms)."""
        from .partition import DECODE

        n = 0
        streams = [pool.phase(DECODE, dm) for dm in
                   (shares or list(range(pool.granularity, pool.n, pool.granularity)) + [pool.n])]
        streams.append(pool.full(0))  # the time-sliced baseline's single stream
        for ps in streams:
            for b in buckets:
                if b <= self.max_batch:
                    self.decode_graph(b, ps)
                    n += 1
        return n

    def stage_decode(self, tokens, ctxs, rows) -> int:
        """Write one decode step's inputs (last token, context incl. it,
        block-table row per request) into pinned staging; pad to the bucket
        with scratch rows (token 0, context 1, page 0).  Returns the bucket."""
        B = len(tokens)
        b = bucket_of(B)
        MP = self.max_pages
        h = self.h_in.numpy()
        tk, cx, bt = h[:b], h[b:2 * b], h[2 * b:2 * b + b * MP].reshape(b, MP)
        tk[:] = 0
        cx[:] = 1
        bt[:] = 0
        tk[:B] = tokens
        cx[:B] = ctxs
        for i, r in enumerate(rows):
            bt[i, :len(r)] = r
        return b

    def launch_decode(self, b: int, ps) -> None:
        """H2D of the staged inputs, the step's graph, D2H of the token ids --
        all on the decode partition's stream (zero-copy kernels)."""
        g = self.decode_graph(b, ps)
        st, MP = ps.torch_stream, self.max_pages
        h = self.h_in
        lib.copy_rows(h[:b].view(1, b), self.d_tok[:b].view(1, b), ps.sms, st)
        lib.copy_rows(h[b:2 * b].view(1, b), self.d_ctx[:b].view(1, b), ps.sms, st)
        lib.copy_rows(h[2 * b:2 * b + b * MP].view(b, MP), self.d_bt[:b], ps.sms, st)
        with torch.cuda.stream(st):  # CUDAGraph.replay launches on the current stream
            g.replay()
        lib.copy_rows(self.d_next[:b].view(1, b), self.h_d_next[:b].view(1, b), ps.sms, st)


class PageAllocator:
    """Free list over the KV pool's pages (page 0 reserved as scratch)."""

    def __init__(self, pages: int):
        self.free = list(range(pages - 1, 0, -1))

    def alloc(self, n: int) -> list[int]:
        if n > len(self.free):
            raise InvalidArgumentError(f"KV pool exhausted: need {n} pages, {len(self.free)} free")
        return [self.free.pop() for _ in range(n)]

    def release(self, pages) -> None:
        self.free.extend(pages)


@dataclass
class _Pending:
    kind: str
    end: torch.cuda.Event
    start: torch.cuda.Event
    payload: dict


def kv_pages_for(cfg: E.SimConfig, max_live_requests: int = 512) -> int:
    """Pages a ServingModel needs so the reference's byte-level KV admission
    (kv_pool_bytes - weights, engine.py:375) can never over-commit it: the
    budget in whole pages plus one partial page per live request, plus the
    scratch page."""
    per_page = kv_bytes(cfg.model, PAGE)
    budget = cfg.kv_pool_bytes - cfg.model.weight_bytes()
    return budget // per_page + max_live_requests + 1


class RealtimeSim(E._ConcurrentSim):
    """`_ConcurrentSim` on a wall clock with the model executing for real
    (module docstring).  Policies: bullet, nopartition, static."""

    def __init__(self, cfg: E.SimConfig, trace, server: ServingModel, pool: PartitionPool, store=None,
                 trace_decisions: bool = False, clock_scale: float = 1.0, prompts=None, seed: int = 0,
                 serialize: bool = False):
        """serialize=True (with policy nopartition): both phases on ONE
        full-device stream -- the time-sliced serving baseline (prefill
        layer steps and decode steps alternate on the device in launch
        order, never concurrently)."""
        if cfg.policy.name == "chunked":
            raise InvalidArgumentError("RealtimeSim runs the concurrent policies; chunked has its own loop")
        if store is None:
            raise InvalidArgumentError("RealtimeSim needs a measured CalibrationStore (no synthetic oracle)")
        super().__init__(cfg, trace, oracle=_NoOracle(), store=store)
        if serialize and cfg.policy.name != "nopartition":
            raise InvalidArgumentError("serialize=True is the time-sliced form of policy nopartition")
        self.serialize = serialize
        self.server = server
        self.pool = pool
        self.pages = PageAllocator(server.kv_pages)
        self.clock_scale = clock_scale
        rng = np.random.default_rng(seed)
        self.prompts = prompts if prompts is not None else {
            r.id: rng.integers(0, server.vocab, r.input_len).astype(np.int32) for r in trace}
        self.seq_pages: dict[int, list[int]] = {}
        self.generated: dict[int, list[int]] = {r.id: [] for r in trace}
        self.last_tok: dict[int, int] = {}
        self.p_pending: _Pending | None = None
        self.d_pending: _Pending | None = None
        self.batch_meta: dict | None = None
        self.trace_decisions = trace_decisions
        self._in_complete = None
        self.decisions: list[dict] = []
        self.host_busy_s = 0.0
        self.device_calls = {"prefill_steps": 0, "decode_steps": 0, "decode_graph_replays": 0}
        # device-timeline gap between a phase's step completing and its next
        # step starting while work was waiting: the control plane's cost
        self.gaps = {"prefill": [], "decode": []}
        self._last_end = {"prefill": None, "decode": None}

    # ------------------------------------------------------------ clock
    def _clock(self) -> float:
        return (time.perf_counter() - self._h0) * self.clock_scale

    def _dev_time(self, ev) -> float:
        return self._t0.elapsed_time(ev) * 1e-3

    # ------------------------------------------------------------- loop
    def run(self) -> E.MetricsReport:
        for r in self.trace:
            self._push(r.arrival_s, "arrival", r.id)
        dev = self.server.dev
        torch.cuda.synchronize(dev)
        self._t0 = _ev()
        self._t0.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        self._h0 = time.perf_counter()
        handlers = {"arrival": self._on_arrival}
        while self.heap or self.p_pending or self.d_pending:
            now = self._clock()
            due = []
            if self.heap and self.heap[0][0] <= now:
                due.append((self.heap[0][0], 0))
            for k, p in ((1, self.p_pending), (2, self.d_pending)):
                if p is not None and p.end.query():
                    due.append((self._dev_time(p.end), k))
            if not due:
                if not self.heap and not (self.p_pending or self.d_pending):
                    break
                _idle(self.heap[0][0] - now if self.heap else None, bool(self.p_pending or self.d_pending))
                continue
            t, k = min(due)
            h0 = time.perf_counter()
            self.now = max(t, 0.0)
            self.makespan = max(self.makespan, t)
            self._apply_partitions(t)
            if k == 0:
                t, _, kind, payload = heapq.heappop(self.heap)
                if kind == "reconfig":
                    self._snapshot(t)
                    if not self.prefill_busy and self.inflight:
                        self._launch_prefill(t)
                    self._maybe_launch_decode(t)
                else:
                    handlers[kind](t, payload)
            elif k == 1:
                p, self.p_pending = self.p_pending, None
                self._in_complete = "prefill"
                self._complete_prefill(t, p)
            else:
                p, self.d_pending = self.d_pending, None
                self._in_complete = "decode"
                self._complete_decode(t, p)
            self._in_complete = None
            self.host_busy_s += time.perf_counter() - h0
        torch.cuda.synchronize(dev)
        self.wall_s = time.perf_counter() - self._h0
        mk = self.makespan
        rep = E.compute_metrics([self.records[r.id] for r in self.trace], self.cfg.slo, mk,
                                self.occ_prefill / mk if mk > 0 else 0.0,
                                self.occ_decode / mk if mk > 0 else 0.0)
        return self._finalize(rep)

    # ------------------------------------------------------ decision log
    def _snapshot_store(self) -> dict:
        s = self.store
        return {"alpha": [[k[0], k[1], k[2], v] for k, v in s.alpha_samples.items()],
                "contention": [[k[0], k[1], v] for k, v in s.contention_bw.items()]}

    def _dynamic_decision(self, t: float) -> list[int]:
        if not self.trace_decisions:
            return super()._dynamic_decision(t)
        state = self._system_state()
        store = self._snapshot_store()
        flags = {"suspended": self.suspended, "in_transition": self.in_transition}
        n_before = len(self.decision_log)
        tasks = super()._dynamic_decision(t)
        entry = self.decision_log[-1] if len(self.decision_log) > n_before else {}
        self.decisions.append({"kind": "prefill", "state": state_to_json(state), "store": store,
                               "flags": flags, "decision": {k: entry.get(k) for k in
                                                            ("pm", "dm", "branch", "batch", "layers")}})
        return tasks

    # ----------------------------------------------------------- prefill
    def _build_batch(self) -> dict:
        """Pages + packed metadata for the newly admitted in-flight batch."""
        srv, dev = self.server, self.server.dev
        toks, pos, slots, cu, last = [], [], [], [0], []
        for rid in self.inflight:
            req = self.records[rid].request
            need = -(-(req.input_len + req.output_len + 1) // PAGE)
            if need > srv.max_pages:
                raise InvalidArgumentError(f"request {rid}: {need} pages exceed max_pages_per_seq")
            pages = self.pages.alloc(need)
            self.seq_pages[rid] = pages
            L = req.input_len
            p = np.arange(L)
            toks.append(self.prompts[rid])
            pos.append(p)
            slots.append(np.asarray(pages, np.int64)[p // PAGE] * PAGE + p % PAGE)
            cu.append(cu[-1] + L)
            last.append(cu[-1] - 1)
        T = cu[-1]
        if T > srv.max_prefill_tokens:
            raise InvalidArgumentError(f"prefill batch of {T} tokens exceeds max_prefill_tokens")

        def d(a, dt=torch.int32):
            return torch.from_numpy(np.ascontiguousarray(np.concatenate(a) if isinstance(a, list) else a)
                                    ).to(dt).to(dev, non_blocking=False)

        return {"T": T, "nseq": len(self.inflight), "max_len": max(np.diff(cu)), "ids": list(self.inflight),
                "tokens": d(toks), "pos": d(pos), "slots": d(slots), "cu": d(np.asarray(cu)),
                "last": d(np.asarray(last), torch.int64)}

    def _launch_prefill(self, t: float) -> None:
        pm = self._prefill_sms_now()
        if pm < 1:
            return
        L = self.model.num_layers
        layers = min(self.cfg.sched.l_step, L - self.layers_done)
        es = ExecutionState(
            prefill_lens=tuple(self.records[r].request.input_len for r in self.inflight),
            prefill_sms=pm,
            decode_ctx_lens=tuple(self.records[r].ctx_len for r in self.decode_running),
            decode_sms=self._decode_sms_now() if self.decode_running else 0)
        if self.layers_done == 0 or self.batch_meta is None or self.batch_meta["ids"] != list(self.inflight):
            self.batch_meta = self._build_batch()
        dm = self._decode_sms_now() if self.decode_running else 0
        ps = (self.pool.full(0) if self.serialize else
              self.pool.split(pm, dm if 0 < dm and pm + dm <= self.n else 0)[0])
        a, b = _ev(), _ev()
        a.record(ps.torch_stream)
        self.server.prefill_layers(self.layers_done, self.layers_done + layers, self.batch_meta, ps.sms,
                                   ps.torch_stream)
        b.record(ps.torch_stream)
        self.prefill_busy = True
        self.device_calls["prefill_steps"] += 1
        self.p_pending = _Pending("prefill", b, a, {"layers": layers, "es": es, "pm": pm,
                                                    "back_to_back": self._in_complete == "prefill"})

    def _gap(self, phase: str, p: _Pending, t_end: float) -> None:
        prev = self._last_end[phase]
        if prev is not None and p.payload.get("back_to_back"):
            self.gaps[phase].append(self._dev_time(p.start) - prev)
        self._last_end[phase] = t_end

    def _complete_prefill(self, t: float, p: _Pending) -> None:
        self._gap("prefill", p, t)
        step_s = p.start.elapsed_time(p.end) * 1e-3
        layers = p.payload["layers"]
        self.occ_prefill += p.payload["pm"] * step_s
        final = self.layers_done + layers >= self.model.num_layers
        if final:
            nxt = self.server.h_p_next[:len(self.inflight)].tolist()
            for rid, tok in zip(self.inflight, nxt):
                self.generated[rid].append(int(tok))
                self.last_tok[rid] = int(tok)
        self._on_prefill_step(t, {"layers": layers, "layer_s": step_s / layers, "es": p.payload["es"]})

    # ------------------------------------------------------------ decode
    def _maybe_launch_decode(self, t: float) -> None:
        """The reference's `_maybe_launch_decode` (engine.py:640-682) with the
        oracle call replaced by the graph-replayed whole-model decode step."""
        if self.decode_busy or self.suspended:
            return
        if not (self.decode_running or self.decode_ready):
            return
        state = self._system_state()
        decision = schedule_decode(state, self.cfg.slo, self.estimator, self.cfg.sched)
        batch = list(decision.next_tasks)
        if self.trace_decisions:
            self.decisions.append({"kind": "decode", "state": state_to_json(state), "store": self._snapshot_store(),
                                   "decision": {"batch": batch, "predicted_step_s": decision.predicted_step_s}})
        if not batch:
            return
        ready = set(self.decode_ready)
        newly = [r for r in batch if r in ready]
        dm = self._decode_sms_now()
        if dm < 1:
            if self.dynamic and self.partition_target[1] < 1:
                from ..scheduler import min_decode_sms

                state.decode_running = tuple(batch)
                state.es = ExecutionState(
                    prefill_lens=state.es.prefill_lens, prefill_sms=state.es.prefill_sms,
                    decode_ctx_lens=tuple(self.records[r].ctx_len for r in batch), decode_sms=0)
                dm_new = min_decode_sms(state, self.cfg.slo, self.estimator, self.cfg.sched)
                if self.inflight or self.queue:
                    dm_new = min(dm_new, self.n - self.cfg.sched.sm_step)
                self._request_partition(t, self.n - dm_new, dm_new)
            return
        for rid in newly:
            self.records[rid].decode_start_s = t
        fresh = set(newly)
        self.decode_ready = [r for r in self.decode_ready if r not in fresh]
        self.decode_running = batch
        pm = self._prefill_sms_now() if self.inflight else 0
        es = ExecutionState(
            prefill_lens=tuple(self.records[r].request.input_len for r in self.inflight),
            prefill_sms=pm,
            decode_ctx_lens=tuple(self.records[r].ctx_len for r in batch),
            decode_sms=dm)
        srv = self.server
        b = srv.stage_decode([self.last_tok[r] for r in batch], [self.records[r].ctx_len for r in batch],
                             [self.seq_pages[r] for r in batch])
        ds = (self.pool.full(0) if self.serialize else
              self.pool.split(pm if 0 < pm and pm + dm <= self.n else 0, dm)[1])
        a, e = _ev(), _ev()
        a.record(ds.torch_stream)
        srv.launch_decode(b, ds)
        e.record(ds.torch_stream)
        self.decode_busy = True
        self.last_decode_event_t = t
        self.device_calls["decode_steps"] += 1
        self.device_calls["decode_graph_replays"] += 1
        self.d_pending = _Pending("decode", e, a, {"batch": batch, "es": es, "dm": dm, "b": len(batch),
                                                   "back_to_back": self._in_complete == "decode"})

    def _complete_decode(self, t: float, p: _Pending) -> None:
        self._gap("decode", p, t)
        step_s = p.start.elapsed_time(p.end) * 1e-3
        self.occ_decode += p.payload["dm"] * step_s
        batch = p.payload["batch"]
        nxt = self.server.h_d_next[:len(batch)].tolist()
        for rid, tok in zip(batch, nxt):
            self.generated[rid].append(int(tok))
            self.last_tok[rid] = int(tok)
        self._on_decode_step(t, {"batch": batch, "step_s": step_s, "es": p.payload["es"]})

    def _finish(self, rid: int) -> None:
        super()._finish(rid)
        pages = self.seq_pages.pop(rid, None)
        if pages:
            self.pages.release(pages)


class _NoOracle:
    """Placeholder for the base class: the device is the oracle here, and any
    call into a synthetic oracle is a bug."""

    def __getattr__(self, name):
        raise InvalidArgumentError(f"RealtimeSim has no synthetic oracle ({name})")


def state_to_json(st) -> dict:
    """A SystemState as plain JSON (the decision-replay fixture format)."""
    es = st.es
    return {"es": {"prefill_lens": list(es.prefill_lens), "prefill_sms": es.prefill_sms,
                   "decode_ctx_lens": list(es.decode_ctx_lens), "decode_sms": es.decode_sms},
            "ps": {"queue": list(st.ps.queue), "in_flight": list(st.ps.in_flight),
                   "layers_done": st.ps.layers_done},
            "requests": [[v.id, v.arrival_s, v.input_len, v.ctx_len] for v in st.requests.values()],
            "sim_time": st.sim_time, "tpot_window": list(st.tpot_window),
            "decode_running": list(st.decode_running), "decode_ready": list(st.decode_ready),
            "kv_blocked": sorted(st.kv_blocked), "decode_last_step_s": st.decode_last_step_s}


def state_from_json(d: dict, mod) -> object:
    """Rebuild a SystemState with module `mod`'s classes (this package's
    scheduler, or the reference's smshare.scheduler / perf_model)."""
    sched, pm = mod
    es = pm.ExecutionState(prefill_lens=tuple(d["es"]["prefill_lens"]), prefill_sms=d["es"]["prefill_sms"],
                           decode_ctx_lens=tuple(d["es"]["decode_ctx_lens"]), decode_sms=d["es"]["decode_sms"])
    reqs = {r[0]: sched.ReqView(r[0], r[1], r[2], r[3]) for r in d["requests"]}
    return sched.SystemState(es=es, ps=sched.PrefillState(list(d["ps"]["queue"]), list(d["ps"]["in_flight"]),
                                                          d["ps"]["layers_done"]),
                             requests=reqs, sim_time=d["sim_time"], tpot_window=tuple(d["tpot_window"]),
                             decode_running=tuple(d["decode_running"]), decode_ready=tuple(d["decode_ready"]),
                             kv_blocked=frozenset(d["kv_blocked"]), decode_last_step_s=d["decode_last_step_s"])


def delta_encode(decisions: list[dict]) -> list[dict]:
    """Fixture compaction: each entry's store snapshot replaced by the alpha
    / contention entries that changed since the previous entry (the first
    entry keeps its full snapshot).  `delta_decode` inverts it."""
    out, prev_a, prev_c = [], {}, {}
    for d in decisions:
        a = {(x[0], x[1], x[2]): x[3] for x in d["store"]["alpha"]}
        c = {(x[0], x[1]): x[2] for x in d["store"]["contention"]}
        da = [[*k, v] for k, v in a.items() if prev_a.get(k) != v]
        dc = [[*k, v] for k, v in c.items() if prev_c.get(k) != v]
        gone = [list(k) for k in prev_a if k not in a] + [list(k) for k in prev_c if k not in c]
        e = dict(d)
        e["store"] = {"alpha": da, "contention": dc, "delta": True, "removed": gone}
        out.append(e)
        prev_a, prev_c = a, c
    return out


def delta_decode(decisions: list[dict]) -> list[dict]:
    out, a, c = [], {}, {}
    for d in decisions:
        st = d["store"]
        if not st.get("delta"):
            out.append(d)
            a = {(x[0], x[1], x[2]): x[3] for x in st["alpha"]}
            c = {(x[0], x[1]): x[2] for x in st["contention"]}
            continue
        for k in st.get("removed", []):
            a.pop(tuple(k), None) if len(k) == 3 else c.pop(tuple(k), None)
        a.update({(x[0], x[1], x[2]): x[3] for x in st["alpha"]})
        c.update({(x[0], x[1]): x[2] for x in st["contention"]})
        e = dict(d)
        e["store"] = {"alpha": [[*k, v] for k, v in a.items()], "contention": [[*k, v] for k, v in c.items()]}
        out.append(e)
    return out


def store_from_json(d: dict, perf_model):
    s = perf_model.CalibrationStore()
    for ph, sms, tok, v in d["alpha"]:
        s.alpha_samples[(ph, int(sms), int(tok))] = v
    for sms, sl, v in d["contention"]:
        s.contention_bw[(int(sms), int(sl))] = v
    return s


class RealtimeChunked(E._ChunkedSim):
    """The reference's lockstep chunked-prefill loop (`_ChunkedSim`,
    engine.py:715-859) on a wall clock, every iteration a real hybrid batch
    through the whole model on the full GPU (the SGLang-style baseline)."""

    def __init__(self, cfg: E.SimConfig, trace, server: ServingModel, pool: PartitionPool, prompts=None,
                 seed: int = 0):
        super().__init__(cfg, trace, oracle=_NoOracle())
        self.server = server
        self.pool = pool
        self.pages = PageAllocator(server.kv_pages)
        rng = np.random.default_rng(seed)
        self.prompts = prompts if prompts is not None else {
            r.id: rng.integers(0, server.vocab, r.input_len).astype(np.int32) for r in trace}
        self.seq_pages: dict[int, list[int]] = {}
        self.generated: dict[int, list[int]] = {r.id: [] for r in trace}
        self.last_tok: dict[int, int] = {}
        self.pending: _Pending | None = None
        self.host_busy_s = 0.0
        self.device_calls = {"hybrid_iterations": 0}

    def run(self) -> E.MetricsReport:
        for r in self.trace:
            self._push(r.arrival_s, "arrival", r.id)
        dev = self.server.dev
        torch.cuda.synchronize(dev)
        self._t0 = _ev()
        self._t0.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        self._h0 = time.perf_counter()
        while self.heap or self.pending:
            now = time.perf_counter() - self._h0
            due = []
            if self.heap and self.heap[0][0] <= now:
                due.append((self.heap[0][0], 0))
            if self.pending is not None and self.pending.end.query():
                due.append((self._t0.elapsed_time(self.pending.end) * 1e-3, 1))
            if not due:
                if not self.heap and not self.pending:
                    break
                _idle(self.heap[0][0] - now if self.heap else None, self.pending is not None)
                continue
            t, k = min(due)
            h0 = time.perf_counter()
            self.makespan = max(self.makespan, t)
            if k == 0:
                t, _, kind, rid = heapq.heappop(self.heap)
                self.queue.append(rid)
                self._log(t)
                if not self.busy:
                    self._start_iteration(t)
            else:
                p, self.pending = self.pending, None
                step_s = p.start.elapsed_time(p.end) * 1e-3
                pl = p.payload
                nxt = self.server.h_p_next[:len(pl["emit_ids"])].tolist()
                for rid, tok in zip(pl["emit_ids"], nxt):
                    self.generated[rid].append(int(tok))
                    self.last_tok[rid] = int(tok)
                tot = pl["chunk_tokens"] + len(pl["decode"])
                if tot > 0:
                    self.occ_prefill += self.gpu.num_sms * step_s * pl["chunk_tokens"] / tot
                    self.occ_decode += self.gpu.num_sms * step_s * len(pl["decode"]) / tot
                self._on_iteration(t, {"chunks": pl["chunks"], "decode": pl["decode"], "step_s": step_s})
            self.host_busy_s += time.perf_counter() - h0
        torch.cuda.synchronize(dev)
        self.wall_s = time.perf_counter() - self._h0
        mk = self.makespan
        rep = E.compute_metrics([self.records[r.id] for r in self.trace], self.cfg.slo, mk,
                                self.occ_prefill / mk if mk > 0 else 0.0,
                                self.occ_decode / mk if mk > 0 else 0.0)
        rep.queue_timeline = self.queue_timeline
        rep.partition_timeline = self.partition_timeline
        rep.decision_log = []
        return rep

    def _start_iteration(self, t: float) -> None:
        """The reference's `_start_iteration` (engine.py:741-800) with the
        oracle replaced by the device iteration."""
        if self.busy:
            return
        for rid in self.decode_ready:
            self.records[rid].decode_start_s = t
        self.decode_running.extend(self.decode_ready)
        self.decode_ready = []
        ds = len(self.decode_running)
        room = max(0, self.cs - ds)
        chunks: list[tuple[int, int, int]] = []
        for rid in self.prefill_fifo:
            if room <= 0:
                break
            left = self.records[rid].request.input_len - self.progress[rid]
            take = min(room, left)
            if take > 0:
                chunks.append((rid, take, self.progress[rid]))
                room -= take
        while room > 0 and self.queue:
            nxt = next((r for r in self.queue if self.kv_used + self._kv_need(r) <= self.kv_budget), None)
            if nxt is None:
                break
            self.queue.remove(nxt)
            self.kv_used += self._kv_need(nxt)
            self.prefill_fifo.append(nxt)
            self.progress[nxt] = 0
            self.records[nxt].state = "prefilling"
            req = self.records[nxt].request
            self.seq_pages[nxt] = self.pages.alloc(-(-(req.input_len + req.output_len + 1) // PAGE))
            take = min(room, req.input_len)
            chunks.append((nxt, take, 0))
            room -= take
        if not chunks and not self.decode_running:
            return
        meta = self._iteration_meta(chunks, list(self.decode_running))
        st = self.pool.full(0)
        a, b = _ev(), _ev()
        a.record(st.torch_stream)
        self.server.hybrid_step(meta, st.sms, st.torch_stream)
        b.record(st.torch_stream)
        self.busy = True
        self.device_calls["hybrid_iterations"] += 1
        self.pending = _Pending("iteration", b, a, {"chunks": chunks, "decode": list(self.decode_running),
                                                    "emit_ids": meta["emit_ids"],
                                                    "chunk_tokens": sum(tk for _, tk, _ in chunks)})

    def _iteration_meta(self, chunks, decode) -> dict:
        srv, dev = self.server, self.server.dev
        MP = srv.max_pages
        n_emit = len(decode) + sum(1 for rid, take, p in chunks if p + take >= self.records[rid].request.input_len)
        if n_emit > srv.max_batch or len(decode) > srv.dsc.max_batch:
            raise InvalidArgumentError(f"hybrid iteration emits {n_emit} rows ({len(decode)} decoding); "
                                       f"the serving model holds {srv.max_batch}")
        toks, pos, slots, emit, emit_ids = [], [], [], [], []
        cu, prior, cbt = [0], [], []
        r = 0
        for rid, take, p in chunks:
            pages = np.asarray(self.seq_pages[rid], np.int64)
            q = np.arange(p, p + take)
            toks.append(self.prompts[rid][p:p + take])
            pos.append(q)
            slots.append(pages[q // PAGE] * PAGE + q % PAGE)
            cu.append(cu[-1] + take)
            prior.append(p)
            row = np.zeros(MP, np.int32)
            row[:len(pages)] = pages
            cbt.append(row)
            r += take
            if p + take >= self.records[rid].request.input_len:
                emit.append(r - 1)
                emit_ids.append(rid)
        Tc = r
        dctx, dbt = [], []
        for rid in decode:
            c = self.records[rid].ctx_len
            pages = np.asarray(self.seq_pages[rid], np.int64)
            toks.append(np.array([self.last_tok[rid]], np.int32))
            pos.append(np.array([c - 1]))
            slots.append(np.array([pages[(c - 1) // PAGE] * PAGE + (c - 1) % PAGE]))
            dctx.append(c)
            row = np.zeros(MP, np.int32)
            row[:len(pages)] = pages
            dbt.append(row)
            emit.append(r)
            emit_ids.append(rid)
            r += 1
        T = r

        def d(a, dt=torch.int32):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

        return {"T": T, "Tc": Tc, "n_chunks": len(chunks), "max_chunk": max([tk for _, tk, _ in chunks] or [1]),
                "tokens": d(np.concatenate(toks)), "pos": d(np.concatenate(pos)), "slots": d(np.concatenate(slots)),
                "cu": d(np.asarray(cu)), "prior": d(np.asarray(prior or [0])),
                "cbt": d(np.stack(cbt) if cbt else np.zeros((1, MP), np.int32)),
                "dctx": d(np.asarray(dctx or [1])), "dbt": d(np.stack(dbt) if dbt else np.zeros((1, MP), np.int32)),
                "emit": d(np.asarray(emit, np.int64), torch.int64), "n_emit": len(emit), "emit_ids": emit_ids}

    def _on_iteration(self, t: float, p: dict) -> None:
        # release the pages of requests this iteration finishes BEFORE the base
        # handler admits new ones (it frees their KV bytes, then starts the
        # next iteration)
        done = [rid for rid in p["decode"]
                if self.records[rid].emitted + 1 >= self.records[rid].request.output_len]
        done += [rid for rid, take, _ in p["chunks"]
                 if self.progress[rid] + take >= self.records[rid].request.input_len
                 and self.records[rid].request.output_len <= 1]
        for rid in done:
            self.pages.release(self.seq_pages.pop(rid))
        super()._on_iteration(t, p)
