"""A whole decoder stack on the B200: embedding, L device layers with their
paged KV caches, final norm and LM head; greedy generation.

Used for BASELINE config 1 (tiny model, token-level parity with the CPU
oracle) and as the model behind the serving driver.  The prefill/decode
launch sequences are DeviceLayer's; this class only threads the residual
stream through the layers and owns the shared paged-KV block pool.
"""

from __future__ import annotations

import torch

from ..workload import ModelSpec
from . import lib
from .layer import (EPS, DecodeScratch, DeviceLayer, KVCache, LayerWeights, PrefillScratch,
                    decode_slots)


class DeviceModel:
    def __init__(self, model: ModelSpec, vocab: int, num_blocks: int, device, seed: int = 0,
                 max_prefill_tokens: int = 4096, max_batch: int = 64, max_pages: int = 256,
                 weights=None, embed=None, final_norm=None, lm_head=None):
        self.model = model
        self.vocab = vocab
        self.device = device
        gen = torch.Generator(device="cpu")
        gen.manual_seed(seed)
        h = model.hidden
        if weights is None:
            weights = [LayerWeights.random(model, device, gen) for _ in range(model.num_layers)]
        self.layers = [DeviceLayer(model, w, device) for w in weights]
        self.rope = self.layers[0].rope
        for lyr in self.layers[1:]:
            lyr.rope = self.rope
        bf = dict(dtype=torch.bfloat16, device=device)
        self.embed = embed if embed is not None else torch.randn(vocab, h, generator=gen).to(**bf)
        self.final_norm = final_norm if final_norm is not None else torch.ones(h, **bf)
        lm_head = lm_head if lm_head is not None else (torch.randn(vocab, h, generator=gen) * 0.05).to(**bf)
        self.lm_head = lib.tile_weight(lm_head)  # streamed by the GEMMs as bulk tiles
        self.caches = [KVCache(num_blocks, model.num_kv_heads, model.head_dim, device)
                       for _ in range(model.num_layers)]
        self.psc = PrefillScratch(model, max_prefill_tokens, device)
        self.dsc = DecodeScratch(model, max_batch, max_pages, device)
        self.buf = [torch.empty(max(max_prefill_tokens, max_batch), h, **bf) for _ in range(2)]
        self.norm_out = torch.empty(max(max_prefill_tokens, max_batch), h, **bf)
        self.logits = torch.empty(max(max_prefill_tokens, max_batch), vocab, **bf)
        self._lm_ws = None
        self._lm_cnt = None

    # --------------------------------------------------------------- passes
    def prefill(self, tokens: torch.Tensor, cu_seqlens: torch.Tensor, max_seqlen: int,
                positions: torch.Tensor, slots: torch.Tensor, sms: int, stream=None,
                hidden_out: list | None = None) -> torch.Tensor:
        """Run all layers over packed prompt tokens; returns the final hidden
        states [T, h] (a view of an internal buffer)."""
        T = tokens.shape[0]
        x = self.buf[0][:T]
        torch.index_select(self.embed, 0, tokens.long(), out=x)
        nseq = cu_seqlens.shape[0] - 1
        for i, (lyr, cache) in enumerate(zip(self.layers, self.caches)):
            y = self.buf[(i + 1) % 2][:T]
            lyr.prefill(x, y, self.psc, cu_seqlens, nseq, max_seqlen, positions, slots, cache, sms, stream)
            if hidden_out is not None:
                hidden_out.append(y.clone())
            x = y
        return x

    def decode(self, tokens: torch.Tensor, ctx_lens: torch.Tensor, block_table: torch.Tensor,
               sms: int, stream=None, hidden_out: list | None = None) -> torch.Tensor:
        """One decode step for B sequences whose newest token is `tokens`
        (already counted in ctx_lens).  Returns final hidden states [B, h]."""
        B = tokens.shape[0]
        pos, slots = decode_slots(block_table, ctx_lens)
        x = self.buf[0][:B]
        torch.index_select(self.embed, 0, tokens.long(), out=x)
        for i, (lyr, cache) in enumerate(zip(self.layers, self.caches)):
            y = self.buf[(i + 1) % 2][:B]
            lyr.decode(x, y, self.dsc, ctx_lens, pos, slots, block_table, cache, sms, stream)
            if hidden_out is not None:
                hidden_out.append(y.clone())
            x = y
        return x

    def hybrid(self, tokens: torch.Tensor, n_chunk_tokens: int, cu_chunks: torch.Tensor, max_chunk: int,
               prior_lens: torch.Tensor, chunk_block_table: torch.Tensor, dec_ctx_lens: torch.Tensor,
               dec_block_table: torch.Tensor, positions: torch.Tensor, slots: torch.Tensor, sms: int,
               stream=None, hidden_out: list | None = None) -> torch.Tensor:
        """One lockstep hybrid iteration through all layers (the chunked-prefill
        baseline, reference _ChunkedSim engine.py:741-800): prefill-chunk rows
        first, then one row per decode sequence.  Returns final hidden [T, h]."""
        T = tokens.shape[0]
        x = self.buf[0][:T]
        torch.index_select(self.embed, 0, tokens.long(), out=x)
        n_chunks = cu_chunks.shape[0] - 1
        for i, (lyr, cache) in enumerate(zip(self.layers, self.caches)):
            y = self.buf[(i + 1) % 2][:T]
            lyr.hybrid(x, y, self.psc, self.dsc, n_chunk_tokens, cu_chunks, n_chunks, max_chunk, prior_lens,
                       chunk_block_table, dec_ctx_lens, dec_block_table, positions, slots, cache, sms, stream)
            if hidden_out is not None:
                hidden_out.append(y.clone())
            x = y
        return x

    def logits_of(self, hidden: torch.Tensor, sms: int, stream=None) -> torch.Tensor:
        n = hidden.shape[0]
        lib.rmsnorm(hidden, self.final_norm, self.norm_out[:n], EPS, sms, stream)
        if n <= 256:
            if self._lm_ws is None:
                nb = max(lib.gemm_swap_ws_bytes(256, self.vocab, self.model.hidden, c) for c in range(1, 149))
                self._lm_ws = torch.empty(nb // 4 + 1, dtype=torch.float32, device=self.device)
                self._lm_cnt = torch.zeros(self.vocab // 128 + 8, dtype=torch.int32, device=self.device)
            lib.gemm_swap(self.norm_out[:n], self.lm_head, self.logits[:n], self._lm_ws, self._lm_cnt,
                          lib.EPI_STORE, max_ctas=sms, stream=stream)
        else:
            lib.gemm(self.norm_out[:n], self.lm_head, self.logits[:n], lib.EPI_STORE, max_ctas=sms,
                     stream=stream)
        return self.logits[:n]
