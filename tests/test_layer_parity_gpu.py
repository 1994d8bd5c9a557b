"""Layer- and model-level parity of the B200 path against the CPU oracle.

Tolerances (see tests/parity_harness.py): |dev - ref| <= 2e-2 + 1e-2 |ref|
on every hidden state; greedy tokens identical at every teacher-forced step
except genuine bf16 ties (top-2 margin within 1 ulp).
"""

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from parity_harness import ATOL, run_llama_hybrid, run_llama_layer, run_tiny, run_tiny_chunked  # noqa: E402


def test_tiny_model_config1_prefill_and_greedy_decode():
    r = run_tiny(seed=0, decode_steps=16)
    assert r["prefill_excess"] <= ATOL, r
    assert r["decode_excess"] <= ATOL, r
    assert r["token_mismatches"] == 0, r
    assert r["tokens_compared"] == r["nseq"] * 17
    assert r["tie_flips"] <= 2, r


def test_llama3_8b_layer_prefill_and_decode():
    r = run_llama_layer(T=512, B=8, ctx=300)
    assert r["prefill_excess"] <= ATOL, r
    assert r["decode_excess"] <= ATOL, r
    assert r["kv_write_max_abs"] <= 2e-2, r


def test_llama3_8b_layer_ragged_prefill_tail():
    # T not a multiple of the 128-row GEMM tile nor of the 64-row attention tile
    r = run_llama_layer(T=333, B=3, ctx=65, seed=3)
    assert r["prefill_excess"] <= ATOL, r
    assert r["decode_excess"] <= ATOL, r


def test_moe_a22b_layer_activated_width():
    # reference MoE preset (workload.py:76-79): 64 q / 4 kv heads of dim 64
    # (GQA 16 -> decode attention head blocks), MLP at 0.1 x 12288 -> 1280 rows
    r = run_llama_layer(T=300, B=5, ctx=200, seed=9, model="moe-a22b")
    assert r["prefill_excess"] <= ATOL, r
    assert r["decode_excess"] <= ATOL, r
    assert r["kv_write_max_abs"] <= 2e-2, r


@pytest.mark.parametrize("budget", [512, 200])
def test_tiny_model_chunked_prefill_hybrid_batches(budget):
    # lockstep hybrid batches (chunks with cached prefixes + decode rows),
    # reference _ChunkedSim engine.py:741-800, hybrid_kernels workload.py:213-257
    r = run_tiny_chunked(seed=0, chunk_budget=budget, decode_steps=6)
    assert r["max_excess"] <= ATOL, r
    assert r["mismatches"] == 0, r
    assert r["chunks_with_prefix"] >= 2 and r["max_chunks_per_iter"] >= 2, r
    assert r["tie_flips"] <= 2, r


def test_llama3_8b_layer_hybrid_batch_with_cached_prefixes():
    r = run_llama_hybrid()
    assert r["excess"] <= ATOL, r
