"""Pin the CPU numerics oracle (oracle/numerics.py) against an independent
implementation of the same layer: Hugging Face transformers'
LlamaDecoderLayer (fp32, eager attention, rotate-half RoPE with theta
500000, RMSNorm eps 1e-5).  The reference (smshare) has no transformer
arithmetic, so this is the oracle's numerics anchor; integer outputs stay
pinned to the reference's own fixtures (tests/golden)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

from oracle import numerics as O  # noqa: E402


def _hf_layer(W, h, Hq, Hkv, d, inter):
    from transformers import LlamaConfig
    from transformers.models.llama.modeling_llama import LlamaDecoderLayer, LlamaRotaryEmbedding

    cfg = LlamaConfig(hidden_size=h, num_attention_heads=Hq, num_key_value_heads=Hkv, head_dim=d,
                      intermediate_size=inter, rms_norm_eps=O.EPS, rope_theta=O.ROPE_THETA,
                      max_position_embeddings=4096, attention_bias=False, mlp_bias=False)
    cfg._attn_implementation = "eager"
    layer = LlamaDecoderLayer(cfg, layer_idx=0).float().eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))  # noqa: E731
    with torch.no_grad():
        layer.self_attn.q_proj.weight.copy_(t(W.w_qkv[: Hq * d]))
        layer.self_attn.k_proj.weight.copy_(t(W.w_qkv[Hq * d:(Hq + Hkv) * d]))
        layer.self_attn.v_proj.weight.copy_(t(W.w_qkv[(Hq + Hkv) * d:]))
        layer.self_attn.o_proj.weight.copy_(t(W.w_o))
        layer.mlp.gate_proj.weight.copy_(t(W.w_gate))
        layer.mlp.up_proj.weight.copy_(t(W.w_up))
        layer.mlp.down_proj.weight.copy_(t(W.w_down))
        layer.input_layernorm.weight.copy_(t(W.attn_norm))
        layer.post_attention_layernorm.weight.copy_(t(W.mlp_norm))
    return layer, LlamaRotaryEmbedding(cfg)


def _run_hf(layer, rope, x, pos):
    T = x.shape[0]
    hs = torch.from_numpy(x.astype(np.float32))[None]
    pid = torch.from_numpy(np.asarray(pos, np.int64))[None]
    cos, sin = rope(hs, pid)
    mask = torch.full((T, T), float("-inf")).triu(1)[None, None]
    with torch.no_grad():
        out = layer(hs, attention_mask=mask, position_ids=pid, position_embeddings=(cos, sin))
    out = out[0] if isinstance(out, tuple) else out
    return out[0].numpy()


@pytest.mark.parametrize("h,Hq,Hkv,d,inter,T,start", [(256, 4, 2, 64, 768, 97, 0), (512, 4, 1, 128, 1024, 64, 300)])
def test_oracle_prefill_layer_matches_hf_llama(h, Hq, Hkv, d, inter, T, start):
    rng = np.random.default_rng(7)
    W = O.LayerWeights(rng.normal(0, 0.02, ((Hq + 2 * Hkv) * d, h)).astype(np.float32),
                       rng.normal(0, 0.02, (h, Hq * d)).astype(np.float32),
                       rng.normal(0, 0.02, (inter, h)).astype(np.float32),
                       rng.normal(0, 0.02, (inter, h)).astype(np.float32),
                       rng.normal(0, 0.02, (h, inter)).astype(np.float32),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32))
    x = rng.normal(size=(T, h)).astype(np.float32)
    pos = np.arange(start, start + T)
    table = O.rope_table(start + T + 1, d)
    ours, _, _ = O.layer_prefill(x, W, Hq, Hkv, d, pos, table, bf16_boundaries=False)
    layer, rope = _hf_layer(W, h, Hq, Hkv, d, inter)
    ref = _run_hf(layer, rope, x, pos)
    assert np.max(np.abs(ours - ref)) < 2e-4 * max(1.0, np.max(np.abs(ref)))


def test_oracle_decode_step_matches_hf_llama_last_row():
    """A decode step over a paged cache filled by the prefill of the first L
    tokens equals the last row of HF's causal layer over all L+1 tokens."""
    h, Hq, Hkv, d, inter, L, page = 256, 4, 2, 64, 512, 150, 64
    rng = np.random.default_rng(11)
    W = O.LayerWeights(rng.normal(0, 0.02, ((Hq + 2 * Hkv) * d, h)).astype(np.float32),
                       rng.normal(0, 0.02, (h, Hq * d)).astype(np.float32),
                       rng.normal(0, 0.02, (inter, h)).astype(np.float32),
                       rng.normal(0, 0.02, (inter, h)).astype(np.float32),
                       rng.normal(0, 0.02, (h, inter)).astype(np.float32),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32),
                       (1 + 0.1 * rng.normal(size=h)).astype(np.float32))
    x = rng.normal(size=(L + 1, h)).astype(np.float32)
    table = O.rope_table(L + 2, d)
    _, k, v = O.layer_prefill(x[:L], W, Hq, Hkv, d, np.arange(L), table, bf16_boundaries=False)
    pages = -(-(L + 1) // page)
    bt = np.array([[5, 2, 7][:pages]], dtype=np.int32)
    kc = np.zeros((8, Hkv, page, d), np.float32)
    vc = np.zeros_like(kc)
    for p in range(L):
        kc[bt[0, p // page], :, p % page] = k[p]
        vc[bt[0, p // page], :, p % page] = v[p]
    ours = O.layer_decode(x[L:], W, Hq, Hkv, d, np.array([L + 1]), table, kc, vc, bt, bf16_boundaries=False)
    layer, rope = _hf_layer(W, h, Hq, Hkv, d, inter)
    ref = _run_hf(layer, rope, x, np.arange(L + 1))[-1:]
    assert np.max(np.abs(ours - ref)) < 2e-4 * max(1.0, np.max(np.abs(ref)))
