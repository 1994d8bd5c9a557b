"""Device-vs-oracle parity harness (TEST INFRASTRUCTURE; used by the gpu tests
and by __graft_entry__.smoke()).

Config 1 of BASELINE.json: a tiny Llama-style model (2 layers, hidden 256, 4
heads of 64, 2 KV heads, intermediate 768, vocab 1024; random init) runs one
1024-token prefill plus 8 requests with contexts {17, 64, 128, 255, 256,
511, 512, 1000} (partial last pages) through the B200 kernels, then 16
greedy decode steps for all 9 sequences, and the same computation in the
numpy oracle (oracle/numerics.py, bf16 rounding at the kernel boundaries).

Tolerances (stated here, asserted by the callers):
  hidden states  |dev - ref| <= ATOL max(1, rms(ref)) + RTOL |ref|  with
                 ATOL = 2e-2, RTOL = 1e-2 (see `excess`; bf16 storage: one ulp
                 at |x| in [4, 8) is 3.1e-2)
  greedy tokens  identical at every step (teacher-forced on the oracle's
                 token, so one near-tie cannot cascade); a difference is
                 tolerated only where the oracle's top-2 logit margin is
                 within MARGIN_ULPS bf16 ulps of the top logit (a genuine
                 bf16 tie) and is reported as `tie_flips`.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import numerics as O  # noqa: E402

ATOL, RTOL = 2e-2, 1e-2
MARGIN_ULPS = 1
TINY_CTX = (17, 64, 128, 255, 256, 511, 512, 1000)
PAGE = 64


def _bf(x):
    return O.bf16_round(np.asarray(x, dtype=np.float32))


def excess(dev, ref) -> float:
    """Normalised tolerance excess: max(|dev-ref| - RTOL|ref|) / max(1, rms(ref)).
    Passing means <= ATOL, i.e. |dev-ref| <= ATOL*max(1, rms(ref)) + RTOL*|ref|
    everywhere: the absolute term scales with the tensor's RMS because
    bf16 rounding differences at the stored intermediates (e.g. SwiGLU
    activations reaching ~25 in a Llama-3-8B layer) propagate in proportion
    to activation scale."""
    dev = np.asarray(dev, np.float32)
    ref = np.asarray(ref, np.float32)
    scale = max(1.0, float(np.sqrt(np.mean(ref.astype(np.float64) ** 2))))
    return float(np.max(np.abs(dev - ref) - RTOL * np.abs(ref))) / scale


def abs_report(dev, ref, tol: float = 2e-2) -> dict:
    """Plain max-abs of dev vs ref against `tol` (north_star: "max-abs
    2e-2"), the share of elements over it, and the bf16 ulp at the tensor's
    peak magnitude.  Both sides store bf16 at the same points, so a 1-ulp
    rounding flip of a stored value |x| in [4, 8) is already 3.1e-2 > tol,
    and flips in h / act propagate through the next 4096- or 14336-deep dot
    product; see DESIGN.md section 5 for the per-tensor accounting."""
    dev = np.asarray(dev, np.float32)
    ref = np.asarray(ref, np.float32)
    diff = np.abs(dev - ref)
    peak = float(np.abs(ref).max()) if ref.size else 0.0
    return {"max_abs": float(diff.max()) if diff.size else 0.0, "tol": tol, "n": int(diff.size),
            "n_over_tol": int((diff > tol).sum()), "frac_over_tol": float((diff > tol).mean()) if diff.size else 0.0,
            "rms_ref": float(np.sqrt(np.mean(ref.astype(np.float64) ** 2))) if ref.size else 0.0,
            "peak_ref": peak, "ulp_at_peak": float(_ulp_bf16(peak)) if peak > 0 else 0.0}


ULP_BUDGET = 2.0


def abs_ok(rep: dict) -> bool:
    """max-abs <= 2e-2, or within ULP_BUDGET bf16 ulps of the tensor's peak
    stored magnitude (one ulp at |x| in [8, 16) is 6.25e-2)."""
    return rep["max_abs"] <= rep["tol"] or rep["max_abs"] <= ULP_BUDGET * rep["ulp_at_peak"]


def tiny_weights(seed: int, vocab: int = 1024):
    from paper_2504_19516_b200.workload import TINY_MODEL as m

    rng = np.random.default_rng(seed)
    h, I = m.hidden, m.intermediate
    layers = []
    for _ in range(m.num_layers):
        layers.append(O.LayerWeights(
            _bf(rng.normal(0, 0.02, (m.qkv_out_dim, h))), _bf(rng.normal(0, 0.02, (h, h))),
            _bf(rng.normal(0, 0.02, (I, h))), _bf(rng.normal(0, 0.02, (I, h))),
            _bf(rng.normal(0, 0.02, (h, I))), _bf(1.0 + 0.1 * rng.normal(size=h)),
            _bf(1.0 + 0.1 * rng.normal(size=h))))
    embed = _bf(rng.normal(0, 1.0, (vocab, h)))
    lm_head = _bf(rng.normal(0, 0.08, (vocab, h)))
    final_norm = _bf(np.ones(h))
    return m, layers, embed, final_norm, lm_head


def _ulp_bf16(x):
    e = np.floor(np.log2(np.maximum(np.abs(x), 1e-30)))
    return 2.0 ** (e - 7)


def run_tiny(seed: int = 0, decode_steps: int = 16, device: int = 0) -> dict:
    """Run config 1 on device and oracle; returns comparison statistics."""
    import torch

    from paper_2504_19516_b200.device.layer import LayerWeights
    from paper_2504_19516_b200.device.model import DeviceModel

    vocab = 1024
    m, Wl, embed, final_norm, lm_head = tiny_weights(seed, vocab)
    dev = torch.device("cuda", device)
    rng = np.random.default_rng(seed + 1)
    prompts = [rng.integers(0, vocab, 1024)] + [rng.integers(0, vocab, c) for c in TINY_CTX]
    lens = [len(p) for p in prompts]
    nseq = len(prompts)
    # paged block pool with a shuffled assignment
    need = [-(-(L + decode_steps + 1) // PAGE) for L in lens]
    nblk = sum(need) + 5
    perm = rng.permutation(nblk)
    max_pages = max(need)
    bt = np.zeros((nseq, max_pages), dtype=np.int32)
    k = 0
    for i, nb in enumerate(need):
        bt[i, :nb] = perm[k:k + nb]
        k += nb

    def t(a, dt=torch.bfloat16):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

    dW = [LayerWeights.from_numpy(dev, w.w_qkv, w.w_o, w.w_gate, w.w_up, w.w_down, w.attn_norm,
                                  w.mlp_norm) for w in Wl]
    dm = DeviceModel(m, vocab, nblk, dev, weights=dW, embed=t(embed), final_norm=t(final_norm),
                     lm_head=t(lm_head), max_prefill_tokens=sum(lens), max_batch=nseq,
                     max_pages=max_pages)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count

    # ---------------- device prefill
    tokens = np.concatenate(prompts).astype(np.int32)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    pos = np.concatenate([np.arange(L) for L in lens]).astype(np.int32)
    slots = np.concatenate([bt[i, np.arange(L) // PAGE] * PAGE + np.arange(L) % PAGE
                            for i, L in enumerate(lens)]).astype(np.int32)
    dev_hidden = []
    hid = dm.prefill(t(tokens, torch.int32), t(cu, torch.int32), max(lens), t(pos, torch.int32),
                     t(slots, torch.int32), sms, hidden_out=dev_hidden)
    last_idx = torch.tensor(cu[1:] - 1, device=dev, dtype=torch.long)
    dev_logits = dm.logits_of(hid[last_idx].contiguous(), sms).float().cpu().numpy()
    dev_hidden = [h.float().cpu().numpy() for h in dev_hidden]

    # ---------------- oracle prefill (per sequence) + cache mirror
    d, Hq, Hkv = m.head_dim, m.num_heads, m.num_kv_heads
    table = O.rope_table(4096, d)
    kc = [np.zeros((nblk, Hkv, PAGE, d), np.float32) for _ in range(m.num_layers)]
    vc = [np.zeros((nblk, Hkv, PAGE, d), np.float32) for _ in range(m.num_layers)]
    ref_hidden = [np.zeros((len(tokens), m.hidden), np.float32) for _ in range(m.num_layers)]
    ref_last = np.zeros((nseq, m.hidden), np.float32)
    for i, p in enumerate(prompts):
        x = embed[p]
        L = len(p)
        for li, W in enumerate(Wl):
            x, kk, vv = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(L), table, bf16_boundaries=True)
            ref_hidden[li][cu[i]:cu[i + 1]] = x
            for j in range(L):
                b, o = bt[i, j // PAGE], j % PAGE
                kc[li][b, :, o, :] = kk[j]
                vc[li][b, :, o, :] = vv[j]
        ref_last[i] = x[-1]

    out = {"prefill_tokens": int(len(tokens)), "nseq": nseq}
    errs = [excess(dev_hidden[li], ref_hidden[li]) for li in range(m.num_layers)]
    out["prefill_max_abs"] = [float(np.max(np.abs(dev_hidden[li] - ref_hidden[li])))
                              for li in range(m.num_layers)]
    out["prefill_abs"] = [abs_report(dev_hidden[li], ref_hidden[li]) for li in range(m.num_layers)]
    out["prefill_excess"] = max(errs)  # <= ATOL required

    # ---------------- greedy decode, teacher-forced on the oracle's tokens
    ref_tok, margin, ref_logits = O.greedy_tokens(ref_last, final_norm, lm_head)
    dev_tok = dev_logits.argmax(-1)
    matches, near_ties, mismatches, tie_flips = 0, 0, 0, 0

    def score(ref_tok, dev_tok, margin, logits):
        nonlocal matches, near_ties, mismatches, tie_flips
        for r, dv, mg, lg in zip(ref_tok, dev_tok, margin, logits):
            tie = mg <= MARGIN_ULPS * _ulp_bf16(np.max(lg))
            near_ties += int(tie)
            if r == dv:
                matches += 1
            elif tie:
                tie_flips += 1
            else:
                mismatches += 1

    score(ref_tok, dev_tok, margin, ref_logits)
    ctx = np.array(lens, dtype=np.int32)
    bt_dev = t(bt, torch.int32)
    cur = ref_tok.astype(np.int32)
    step_err, step_abs = [], []
    for s in range(decode_steps):
        ctx = ctx + 1
        hid = dm.decode(t(cur, torch.int32), t(ctx, torch.int32), bt_dev, sms)
        dl = dm.logits_of(hid, sms).float().cpu().numpy()
        dh = hid.float().cpu().numpy()
        x = embed[cur]
        for li, W in enumerate(Wl):
            x = O.layer_decode(x, W, Hq, Hkv, d, ctx, table, kc[li], vc[li], bt, bf16_boundaries=True)
        step_err.append(excess(dh, x))
        step_abs.append(abs_report(dh, x))
        rt, mg, lg = O.greedy_tokens(x, final_norm, lm_head)
        score(rt, dl.argmax(-1), mg, lg)
        cur = rt.astype(np.int32)
    out["decode_excess"] = max(step_err)
    out["decode_max_abs"] = max(a["max_abs"] for a in step_abs)
    out["decode_abs_ok"] = all(abs_ok(a) for a in step_abs)
    out["tokens_compared"] = matches + mismatches + tie_flips
    out["token_matches"] = matches
    out["token_mismatches"] = mismatches
    out["near_ties"] = near_ties
    out["tie_flips"] = tie_flips
    return out


def run_llama_layer(T: int = 512, B: int = 8, ctx: int = 300, seed: int = 0, device: int = 0,
                    model: str = "llama3-8b") -> dict:
    """Config-2 numerics at a CPU-affordable size: one layer of a reference
    preset (default Llama-3-8B; moe-a22b at its activated MLP width), prefill
    of T tokens and one decode step for B sequences of context ctx, device vs
    oracle."""
    import torch

    from paper_2504_19516_b200.device.layer import (DecodeScratch, DeviceLayer, KVCache,
                                                    LayerWeights, PrefillScratch, decode_slots, mlp_width)
    from paper_2504_19516_b200.workload import MODEL_PRESETS

    m = MODEL_PRESETS[model]
    rng = np.random.default_rng(seed)
    h, I, d, Hq, Hkv = m.hidden, mlp_width(m), m.head_dim, m.num_heads, m.num_kv_heads
    W = O.LayerWeights(_bf(rng.normal(0, 0.02, (m.qkv_out_dim, h))), _bf(rng.normal(0, 0.02, (h, h))),
                       _bf(rng.normal(0, 0.02, (I, h))), _bf(rng.normal(0, 0.02, (I, h))),
                       _bf(rng.normal(0, 0.02, (h, I))), _bf(1 + 0.1 * rng.normal(size=h)),
                       _bf(1 + 0.1 * rng.normal(size=h)))
    dev = torch.device("cuda", device)
    lyr = DeviceLayer(m, LayerWeights.from_numpy(dev, W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down,
                                                 W.attn_norm, W.mlp_norm), dev, max_pos=max(T, ctx) + 2)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    table = O.rope_table(max(T, ctx) + 2, d)

    def t(a, dt=torch.bfloat16):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

    # prefill
    x = _bf(rng.normal(size=(T, h)))
    cache = KVCache(-(-T // PAGE), Hkv, d, dev)
    y = torch.empty(T, h, dtype=torch.bfloat16, device=dev)
    lyr.prefill(t(x), y, PrefillScratch(m, T, dev), t(np.array([0, T]), torch.int32), 1, T,
                t(np.arange(T), torch.int32), t(np.arange(T), torch.int32), cache, sms)
    ref, _, _ = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(T), table, bf16_boundaries=True)
    dy = y.float().cpu().numpy()
    res = {"prefill_max_abs": float(np.max(np.abs(dy - ref))), "prefill_excess": excess(dy, ref)}
    # decode: B sequences with random cache contents, one new token each
    pages = -(-(ctx) // PAGE)
    nblk = B * pages + 3
    kc = _bf(rng.normal(size=(nblk, Hkv, PAGE, d)))
    vc = _bf(rng.normal(size=(nblk, Hkv, PAGE, d)))
    bt = rng.permutation(nblk)[: B * pages].reshape(B, pages).astype(np.int32)
    ctxs = np.array([ctx - 7 * i for i in range(B)], dtype=np.int32)
    xd = _bf(rng.normal(size=(B, h)))
    dcache = KVCache(nblk, Hkv, d, dev)
    from paper_2504_19516_b200.device import lib

    dcache.k.copy_(lib.kv_pack(t(kc)))
    dcache.v.copy_(lib.kv_pack(t(vc)))
    ctx_t, bt_t = t(ctxs, torch.int32), t(bt, torch.int32)
    pos, slots = decode_slots(bt_t, ctx_t)
    yd = torch.empty(B, h, dtype=torch.bfloat16, device=dev)
    lyr.decode(t(xd), yd, DecodeScratch(m, B, pages, dev), ctx_t, pos, slots, bt_t, dcache, sms)
    refd = O.layer_decode(xd, W, Hq, Hkv, d, ctxs, table, kc, vc, bt, bf16_boundaries=True)
    dyd = yd.float().cpu().numpy()
    res["decode_max_abs"] = float(np.max(np.abs(dyd - refd)))
    res["decode_excess"] = excess(dyd, refd)
    # the new tokens' K/V landed in the cache slots
    kdev = lib.kv_unpack(dcache.k).float().cpu().numpy()
    res["kv_write_max_abs"] = float(max(np.max(np.abs(kdev[bt[b, (c - 1) // PAGE], :, (c - 1) % PAGE] -
                                                      kc[bt[b, (c - 1) // PAGE], :, (c - 1) % PAGE]))
                                        for b, c in enumerate(ctxs)))
    return res


def run_tiny_chunked(seed: int = 0, chunk_budget: int = 512, decode_steps: int = 6, device: int = 0) -> dict:
    """Config 1 through the lockstep chunked-prefill path (hybrid batches,
    reference _ChunkedSim engine.py:741-800 / hybrid_kernels workload.py:
    213-257) on the device vs the oracle's `layer_hybrid`.

    The 9 prompts of `run_tiny` are admitted FIFO; every iteration packs the
    running decode tokens first, then prompt chunks up to `chunk_budget`
    tokens (so chunks carry cached prefixes and several sequences share an
    iteration).  A prompt's completion emits its greedy token (teacher-forced
    on the oracle's) and the sequence decodes `decode_steps` more tokens."""
    import torch

    from paper_2504_19516_b200.device.layer import LayerWeights
    from paper_2504_19516_b200.device.model import DeviceModel

    vocab = 1024
    m, Wl, embed, final_norm, lm_head = tiny_weights(seed, vocab)
    dev = torch.device("cuda", device)
    rng = np.random.default_rng(seed + 1)
    prompts = [rng.integers(0, vocab, 1024)] + [rng.integers(0, vocab, c) for c in TINY_CTX]
    lens = [len(p) for p in prompts]
    nseq = len(prompts)
    need = [-(-(L + decode_steps + 2) // PAGE) for L in lens]
    nblk = sum(need) + 5
    perm = rng.permutation(nblk)
    max_pages = max(need)
    bt = np.zeros((nseq, max_pages), dtype=np.int32)
    k = 0
    for i, nb in enumerate(need):
        bt[i, :nb] = perm[k:k + nb]
        k += nb

    def t(a, dt=torch.bfloat16):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

    dW = [LayerWeights.from_numpy(dev, w.w_qkv, w.w_o, w.w_gate, w.w_up, w.w_down, w.attn_norm,
                                  w.mlp_norm) for w in Wl]
    dm = DeviceModel(m, vocab, nblk, dev, weights=dW, embed=t(embed), final_norm=t(final_norm),
                     lm_head=t(lm_head), max_prefill_tokens=chunk_budget, max_batch=nseq,
                     max_pages=max_pages)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    d, Hq, Hkv = m.head_dim, m.num_heads, m.num_kv_heads
    table = O.rope_table(4096, d)
    kc = [np.zeros((nblk, Hkv, PAGE, d), np.float32) for _ in range(m.num_layers)]
    vc = [np.zeros((nblk, Hkv, PAGE, d), np.float32) for _ in range(m.num_layers)]

    progress = [0] * nseq
    queue = list(range(nseq))
    running: list[int] = []       # decoding sequences
    ctx = [0] * nseq              # tokens in cache incl. the pending one (decoders)
    last_tok = [0] * nseq
    emitted = [0] * nseq
    stats = {"iterations": 0, "max_chunks_per_iter": 0, "chunks_with_prefix": 0, "excess": [],
             "matches": 0, "mismatches": 0, "tie_flips": 0, "near_ties": 0}
    while queue or running:
        dec = list(running)
        budget = chunk_budget - len(dec)
        chunks = []  # (seq, take, prior)
        for sid in list(queue):
            if budget <= 0:
                break
            take = min(budget, lens[sid] - progress[sid])
            chunks.append((sid, take, progress[sid]))
            budget -= take
        toks = [prompts[s][p:p + n] for s, n, p in chunks] + [np.array([last_tok[s]]) for s in dec]
        tokens = np.concatenate(toks).astype(np.int32)
        seqs = [(n, p) for _, n, p in chunks] + [(1, ctx[s] - 1) for s in dec]
        rows_bt = bt[[s for s, _, _ in chunks] + dec]
        pos = np.concatenate([np.arange(p, p + n) for n, p in seqs]).astype(np.int32)
        slots = np.concatenate([rows_bt[i, np.arange(p, p + n) // PAGE] * PAGE + np.arange(p, p + n) % PAGE
                                for i, (n, p) in enumerate(seqs)]).astype(np.int32)
        Tc = sum(n for _, n, _ in chunks)
        cu = np.concatenate([[0], np.cumsum([n for _, n, _ in chunks])]).astype(np.int32)
        prior = np.array([p for _, _, p in chunks] or [0], dtype=np.int32)
        cbt = bt[[s for s, _, _ in chunks]] if chunks else bt[:1]
        dbt = bt[dec] if dec else bt[:1]
        dctx = np.array([ctx[s] for s in dec] or [1], dtype=np.int32)
        hid = dm.hybrid(t(tokens, torch.int32), Tc, t(cu, torch.int32), max([n for _, n, _ in chunks] or [1]),
                        t(prior, torch.int32), t(cbt, torch.int32), t(dctx, torch.int32), t(dbt, torch.int32),
                        t(pos, torch.int32), t(slots, torch.int32), sms)
        dh = hid.float().cpu().numpy()
        x = embed[tokens]
        for li, W in enumerate(Wl):
            x = O.layer_hybrid(x, W, Hq, Hkv, d, seqs, table, kc[li], vc[li], rows_bt, bf16_boundaries=True)
        stats["excess"].append(excess(dh, x))
        stats["iterations"] += 1
        stats["max_chunks_per_iter"] = max(stats["max_chunks_per_iter"], len(chunks))
        stats["chunks_with_prefix"] += sum(1 for _, _, p in chunks if p > 0)
        # rows whose next token is sampled: completed prompts and decoders
        emit_rows, emit_seqs = [], []
        r = 0
        for s, n, p in chunks:
            r += n
            progress[s] += n
            if progress[s] == lens[s]:
                emit_rows.append(r - 1)
                emit_seqs.append(s)
                queue.remove(s)
        for j, s in enumerate(dec):
            emit_rows.append(Tc + j)
            emit_seqs.append(s)
        if emit_rows:
            idx = torch.tensor(emit_rows, device=dev, dtype=torch.long)
            dl = dm.logits_of(hid[idx].contiguous(), sms).float().cpu().numpy()
            rt, mg, lg = O.greedy_tokens(x[emit_rows], final_norm, lm_head)
            for rr, dv, g, l in zip(rt, dl.argmax(-1), mg, lg):
                tie = g <= MARGIN_ULPS * _ulp_bf16(np.max(l))
                stats["near_ties"] += int(tie)
                if rr == dv:
                    stats["matches"] += 1
                elif tie:
                    stats["tie_flips"] += 1
                else:
                    stats["mismatches"] += 1
            for s, tok in zip(emit_seqs, rt):
                last_tok[s] = int(tok)
                emitted[s] += 1
                if s not in running:
                    running.append(s)
                    ctx[s] = lens[s] + 1
                else:
                    ctx[s] += 1
        running = [s for s in running if emitted[s] <= decode_steps]
    stats["max_excess"] = max(stats["excess"])
    del stats["excess"]
    return stats


def run_llama_hybrid(seed: int = 5, device: int = 0) -> dict:
    """One Llama-3-8B layer over a hybrid batch at full width: two prompt
    chunks with cached prefixes (priors 0 and 700) plus 5 decode rows, device
    (DeviceLayer.hybrid: GEMMs over the concatenated rows, paged prefill
    attention, paged decode attention) vs oracle `layer_hybrid`."""
    import torch

    from paper_2504_19516_b200.device import lib
    from paper_2504_19516_b200.device.layer import (DecodeScratch, DeviceLayer, KVCache, LayerWeights,
                                                    PrefillScratch)
    from paper_2504_19516_b200.workload import MODEL_PRESETS

    m = MODEL_PRESETS["llama3-8b"]
    rng = np.random.default_rng(seed)
    h, I, d, Hq, Hkv = m.hidden, m.intermediate, m.head_dim, m.num_heads, m.num_kv_heads
    W = O.LayerWeights(_bf(rng.normal(0, 0.02, (m.qkv_out_dim, h))), _bf(rng.normal(0, 0.02, (h, h))),
                       _bf(rng.normal(0, 0.02, (I, h))), _bf(rng.normal(0, 0.02, (I, h))),
                       _bf(rng.normal(0, 0.02, (h, I))), _bf(1 + 0.1 * rng.normal(size=h)),
                       _bf(1 + 0.1 * rng.normal(size=h)))
    dev = torch.device("cuda", device)
    seqs = [(200, 0), (130, 700)] + [(1, c - 1) for c in (65, 300, 1000, 64, 129)]
    nseq = len(seqs)
    pages = [-(-(n + p) // PAGE) for n, p in seqs]
    nblk = sum(pages) + 3
    perm = rng.permutation(nblk)
    bt = np.zeros((nseq, max(pages)), np.int32)
    k = 0
    for i, pg in enumerate(pages):
        bt[i, :pg] = perm[k:k + pg]
        k += pg
    # cached prefixes: random K/V (bf16 values) in every page, identical on both sides
    kc = _bf(rng.normal(size=(nblk, Hkv, PAGE, d)))
    vc = _bf(rng.normal(size=(nblk, Hkv, PAGE, d)))
    T = sum(n for n, _ in seqs)
    x = _bf(rng.normal(size=(T, h)))
    table = O.rope_table(2048, d)

    def t(a, dt=torch.bfloat16):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dt).to(dev)

    lyr = DeviceLayer(m, LayerWeights.from_numpy(dev, W.w_qkv, W.w_o, W.w_gate, W.w_up, W.w_down, W.attn_norm,
                                                 W.mlp_norm), dev, max_pos=2048)
    cache = KVCache(nblk, Hkv, d, dev)
    cache.k.copy_(lib.kv_pack(t(kc)))
    cache.v.copy_(lib.kv_pack(t(vc)))
    nc = 2
    Tc = seqs[0][0] + seqs[1][0]
    pos = np.concatenate([np.arange(p, p + n) for n, p in seqs]).astype(np.int32)
    slots = np.concatenate([bt[i, np.arange(p, p + n) // PAGE] * PAGE + np.arange(p, p + n) % PAGE
                            for i, (n, p) in enumerate(seqs)]).astype(np.int32)
    y = torch.empty(T, h, dtype=torch.bfloat16, device=dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    lyr.hybrid(t(x), y, PrefillScratch(m, T, dev), DecodeScratch(m, nseq - nc, max(pages), dev), Tc,
               t(np.array([0, seqs[0][0], Tc]), torch.int32), nc, max(seqs[0][0], seqs[1][0]),
               t(np.array([0, 700]), torch.int32), t(bt[:nc], torch.int32),
               t(np.array([p + 1 for _, p in seqs[nc:]]), torch.int32), t(bt[nc:], torch.int32),
               t(pos, torch.int32), t(slots, torch.int32), cache, sms)
    ref = O.layer_hybrid(x, W, Hq, Hkv, d, seqs, table, kc, vc, bt, bf16_boundaries=True)
    dy = y.float().cpu().numpy()
    return {"max_abs": float(np.max(np.abs(dy - ref))), "excess": excess(dy, ref),
            "chunk_excess": excess(dy[:Tc], ref[:Tc]), "decode_excess": excess(dy[Tc:], ref[Tc:])}


def groups_teacher_forced(W, x, attn_ref, dev: dict, y_dev) -> dict:
    """Each kernel group of the layer (workload.py:162-210) re-run by the
    oracle on the DEVICE's own bf16 input to that group, so a group's error
    is its own and not inherited through earlier bf16 rounding flips:
      attn         attention over the device's q / k / v  -> device attn
      o_proj       x + attn_dev . W_o^T                   -> device h
      mlp_up_gate  silu(n(h_dev) W_g^T) * (n(h_dev) W_u^T) -> device act
      mlp_down     h_dev + act_dev . W_down^T             -> device y
    (`attn_ref` is the oracle attention over the device's q/k/v.)"""
    b = O.bf16_round
    n2 = b(O.rmsnorm(dev["h"], W.mlp_norm))
    ref = {"attn": b(attn_ref.reshape(dev["attn"].shape)),
           "o_proj": b(x + dev["attn"] @ W.w_o.T),
           "mlp_up_gate": b(O.silu(n2 @ W.w_gate.T) * (n2 @ W.w_up.T)),
           "mlp_down": b(dev["h"] + dev["act"] @ W.w_down.T)}
    got = {"attn": dev["attn"], "o_proj": dev["h"], "mlp_up_gate": dev["act"], "mlp_down": y_dev}
    return {g: dict(abs_report(got[g], ref[g]), excess=excess(got[g], ref[g])) for g in ref}


def run_corun_parity(T: int = 4096, dm: int = 8, B: int = 32, ctx: int = 2048, n_decode: int | None = None,
                     seed: int = 21, device: int = 0, model: str = "llama3-8b") -> dict:
    """BASELINE config 2 at the benchmarked size, under co-execution: one
    Llama-3-8B layer's prefill over T tokens on a (N - dm)-SM green context
    WHILE the decode layer-step's CUDA graph (B sequences of context ctx,
    paged KV) replays on the dm-SM side -- the exact launch sequence of
    bench.py's timed region (CoRunner.corun).  Both outputs, and the prefill's
    paged K/V writes, are compared with the numpy oracle (workload.py:162-210
    decomposition).  Weights N(0, 0.02), activations and caches N(0, 1), all
    drawn on the device from a seeded generator and copied to the oracle."""
    import torch

    from paper_2504_19516_b200.device import lib
    from paper_2504_19516_b200.device.corun import CoRunner
    from paper_2504_19516_b200.device.layer import LayerWeights, mlp_width
    from paper_2504_19516_b200.device.partition import DECODE, PREFILL
    from paper_2504_19516_b200.workload import MODEL_PRESETS

    m = MODEL_PRESETS[model]
    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    h, I, d, Hq, Hkv = m.hidden, mlp_width(m), m.head_dim, m.num_heads, m.num_kv_heads
    bf = torch.bfloat16

    def w(*shape, std=0.02):
        return (torch.randn(*shape, generator=g, device=dev) * std).to(bf)

    dense = [w(m.qkv_out_dim, h), w(h, h), w(I, h), w(I, h), w(h, I),
             (1 + 0.1 * torch.randn(h, generator=g, device=dev)).to(bf),
             (1 + 0.1 * torch.randn(h, generator=g, device=dev)).to(bf)]
    cr = CoRunner(m, T, B, ctx, device=device, seed=seed, weights=LayerWeights.from_dense(*dense))
    pages = -(-ctx // PAGE)
    nblk = B * pages
    kc, vc = w(nblk, Hkv, PAGE, d, std=1.0), w(nblk, Hkv, PAGE, d, std=1.0)
    px, dx = w(T, h, std=1.0), w(B, h, std=1.0)
    cr.load(px=px, dx=dx, kcache=kc, vcache=vc)
    N = cr.n
    pm = N - dm
    if n_decode is None:  # enough decode steps to cover the prefill layer
        n_decode = max(1, round(cr.isolated(PREFILL, pm, reps=2) / cr.isolated(DECODE, dm, reps=2)))
    res = cr.corun(pm, dm, 1, n_decode)
    torch.cuda.synchronize()
    py = cr.py.float().cpu().numpy()
    dy = cr.dy.float().cpu().numpy()
    pk = lib.kv_unpack(cr.pcache.k).float().cpu().numpy()
    pv = lib.kv_unpack(cr.pcache.v).float().cpu().numpy()
    bt = cr.block_table.cpu().numpy()

    def f(t):
        return t.float().cpu().numpy()

    W = O.LayerWeights(*[f(t) for t in dense])
    table = O.rope_table(max(T, ctx) + 1, d)
    tr_p, tr_d = {}, {}
    xin_p, xin_d = f(px), f(dx)
    ref_p, k_rot, v_ref = O.layer_prefill(xin_p, W, Hq, Hkv, d, np.arange(T), table, bf16_boundaries=True,
                                          trace=tr_p)
    kc_np, vc_np = f(kc), f(vc)
    ref_d = O.layer_decode(xin_d, W, Hq, Hkv, d, np.full(B, ctx), table, kc_np, vc_np, bt,
                           bf16_boundaries=True, trace=tr_d)
    # prefill K/V: slot t -> block t // 64 (CoRunner's identity slots)
    pk_t = pk.transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:T]
    pv_t = pv.transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:T]
    # per-tensor parity of the stored intermediates (q after RoPE, attention
    # output, residual h after o_proj, SwiGLU act) and the layer outputs
    Hqd = Hq * d
    dev_p = {"q": cr.psc.qkv[:T, :Hqd], "attn": cr.psc.attn[:T], "h": cr.psc.h[:T], "act": cr.psc.act[:T]}
    dev_d = {"q": cr.dsc.qkv[:B, :Hqd], "attn": cr.dsc.attn[:B], "h": cr.dsc.h[:B], "act": cr.dsc.act[:B]}
    scale = 1.0 / math.sqrt(d)
    Hkd = Hkv * d
    qkv_p = f(cr.psc.qkv[:T])
    att_p = O.causal_attention(qkv_p[:, :Hqd].reshape(T, Hq, d), qkv_p[:, Hqd:Hqd + Hkd].reshape(T, Hkv, d),
                               qkv_p[:, Hqd + Hkd:].reshape(T, Hkv, d), scale)
    kc_dev = lib.kv_unpack(cr.dcache.k[:nblk]).float().cpu().numpy()
    vc_dev = lib.kv_unpack(cr.dcache.v[:nblk]).float().cpu().numpy()
    att_d = O.paged_decode_attention(f(cr.dsc.qkv[:B, :Hqd]).reshape(B, Hq, d), kc_dev, vc_dev, bt,
                                     np.full(B, ctx), scale)
    del kc_dev, vc_dev
    out = {"T": T, "pm": pm, "dm": dm, "B": B, "ctx": ctx, "decode_steps": n_decode,
           "prefill_groups": groups_teacher_forced(W, xin_p, att_p, {k: f(v) for k, v in dev_p.items()}, py),
           "decode_groups": groups_teacher_forced(W, xin_d, att_d, {k: f(v) for k, v in dev_d.items()}, dy),
           "prefill_s": res.prefill_layer_s[0], "decode_s": res.decode_layer_s,
           "span_s": res.span_s, "overlap_s": res.overlap_s(),
           "prefill_abs": abs_report(py, ref_p), "prefill_excess": excess(py, ref_p),
           "decode_abs": abs_report(dy, ref_d), "decode_excess": excess(dy, ref_d),
           "kv_k_abs": abs_report(pk_t, O.bf16_round(k_rot)), "kv_v_abs": abs_report(pv_t, O.bf16_round(v_ref)),
           "prefill_tensors": {k: dict(abs_report(f(v), tr_p[k]), excess=excess(f(v), tr_p[k]))
                               for k, v in dev_p.items()},
           "decode_tensors": {k: dict(abs_report(f(v), tr_d[k]), excess=excess(f(v), tr_d[k]))
                              for k, v in dev_d.items()}}
    return out


def oracle_check_generation(m, Wl, embed, final_norm, lm_head, prompt, tokens) -> dict:
    """Teacher-force the oracle on a sequence the DEVICE generated freely
    (prompt, then its greedy tokens): at every step the device's token must
    be the oracle's argmax, or a genuine bf16 tie (top-2 margin within
    MARGIN_ULPS ulps of the top logit)."""
    d, Hq, Hkv = m.head_dim, m.num_heads, m.num_kv_heads
    L, n = len(prompt), len(tokens)
    pages = -(-(L + n + 1) // PAGE)
    kc = [np.zeros((pages, Hkv, PAGE, d), np.float32) for _ in Wl]
    vc = [np.zeros((pages, Hkv, PAGE, d), np.float32) for _ in Wl]
    bt = np.arange(pages, dtype=np.int32)[None]
    table = O.rope_table(L + n + 2, d)
    out = {"matches": 0, "mismatches": 0, "tie_flips": 0, "first_bad": None}

    def score(i, x):
        rt, mg, lg = O.greedy_tokens(x, final_norm, lm_head)
        if int(rt[0]) == int(tokens[i]):
            out["matches"] += 1
        elif mg[0] <= MARGIN_ULPS * _ulp_bf16(np.max(lg[0])):
            out["tie_flips"] += 1
        else:
            out["mismatches"] += 1
            if out["first_bad"] is None:
                out["first_bad"] = i

    x = embed[np.asarray(prompt)]
    for li, W in enumerate(Wl):
        x, kk, vv = O.layer_prefill(x, W, Hq, Hkv, d, np.arange(L), table, bf16_boundaries=True)
        for j in range(L):
            kc[li][j // PAGE, :, j % PAGE] = kk[j]
            vc[li][j // PAGE, :, j % PAGE] = vv[j]
    score(0, x[-1:])
    for i in range(1, n):
        x = embed[[int(tokens[i - 1])]]
        for li, W in enumerate(Wl):
            x = O.layer_decode(x, W, Hq, Hkv, d, np.array([L + i]), table, kc[li], vc[li], bt,
                               bf16_boundaries=True)
        score(i, x)
    return out
