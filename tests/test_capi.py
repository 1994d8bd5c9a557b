"""The C-ABI library loads on a GPU-less host and exports every symbol that
include/hp.h declares; host-only entry points behave (no compute calls)."""

import re
from pathlib import Path

import pytest

from paper_2504_19516_b200.device import lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "hp.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    so = lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(so, s), f"{s} declared in hp.h but not exported"
    # and the ctypes signature table covers exactly the header
    assert set(lib.SIGNATURES) == set(syms)


def test_abi_version_and_device_count():
    so = lib.load()
    assert so.hp_abi_version() == 1
    assert so.hp_device_count() >= 0


def test_wave_stats_host_entry_point():
    assert lib.wave_stats(216, 2, 108) == (1, 108, 0.0)
    assert lib.wave_stats(110, 1, 108) == (2, 2, 106 / 216)
    assert lib.wave_stats(384, 1, 108) == (4, 60, 48 / 432)
    with pytest.raises(ValueError, match="positive"):
        lib.wave_stats(0, 1, 148)


def test_invalid_arguments_are_rejected_before_any_launch():
    so = lib.load()
    # null pointers / bad shapes fail with HP_ERR_INVALID and a message
    rc = so.hp_gemm(None, 0, None, 0, None, 0, None, 0, 128, 128, 64, 0, 148, None)
    assert rc == -1
    assert b"null" in so.hp_last_error()
    rc = so.hp_decode_attn(1, 128, 1, 1, 1, 1, 1, 1, 128, 1, 4, 1, 96, 64, 1, 0.1, None, 0, 1, None)
    assert rc == -1 and b"head_dim" in so.hp_last_error()


def test_workspace_sizing_is_host_side():
    n = lib.gemm_swap_ws_bytes(32, 4096, 4096, 148)
    assert n > 0 and n % 4 == 0
    assert lib.decode_attn_ws_bytes(32, 32, 128, 4) == 32 * 32 * 4 * 130 * 4


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(lib, "_LIB", None)
    with pytest.raises(lib.HotPathError, match="no CPU fallback"):
        lib.load(tmp_path / "nope.so")


def test_gemm_tile_planner_is_host_side():
    # hp_gemm_plan: CTA-pair 256x256 tiles by default (the stream-K tail
    # absorbs the last round); without the tail, 128-wide single-CTA tiles
    # where they save a wave-quantised round (T=1024 qkv on 148 SMs)
    assert lib.gemm_plan(4096, 28672, 4096, 140) == (256, 16 * 112, 2)
    assert lib.gemm_plan(4096, 4096, 4096, 140) == (256, 16 * 16, 2)
    bn, tiles, cpt = lib.gemm_plan(1024, 6144, 4096, 148)
    assert (bn, cpt) == (128, 1) and tiles == 8 * 48
    # the stream-K tail only for long-K GEMMs whose last round would leave
    # >= half the pairs idle: T = 1024 mlp_down on 124 SMs (64 tiles, 62
    # pairs) runs as pair tiles with the last two rounds split evenly
    assert lib.gemm_plan(1024, 4096, 14336, 124) == (256, 4 * 16, 2)
    assert lib.gemm_tail_tiles(1024, 4096, 14336, 124) == 64
    assert lib.gemm_tail_tiles(4096, 4096, 14336, 140) == 0  # 256 = 3 x 70 + 46: plain
    assert lib.gemm_tail_tiles(4096, 4096, 4096, 148) == 0   # short K: plain
    lib.set_gemm_tail(0)
    try:
        assert lib.gemm_tail_tiles(1024, 4096, 14336, 124) == 0
        assert lib.gemm_plan(1024, 4096, 14336, 124)[2] == 1  # plain: 128-wide single-CTA tiles
    finally:
        lib.set_gemm_tail(-1)
    assert lib.gemm_plan(300, 512, 640, 1)[2] == 1  # one SM: no pair
    from paper_2504_19516_b200.perf_model import wave_stats

    # the rounds the persistent grid runs are the paper's wave count
    _, t, c = lib.gemm_plan(4096, 6144, 4096, 140)
    assert wave_stats(t, 1, 140 // c).waves == 6


def test_decode_attention_launch_count_is_host_side():
    # one launch while the context is not split, a combine launch otherwise
    assert lib.decode_attn_launches(32, 32, 8, 128, 32, 64, 8) == 1
    assert lib.decode_attn_launches(32, 32, 8, 128, 32, 64, 148) == 1  # 256 units >= 148 / 2: no split
    assert lib.decode_attn_launches(4, 32, 8, 128, 32, 64, 148) == 2   # 32 units: split + combine
    assert lib.decode_attn_launches(0, 32, 8, 128, 32, 64, 148) == 0
    assert lib.decode_attn_launches(32, 64, 4, 64, 32, 64, 148) == 1  # moe-a22b: 128 units
    assert lib.decode_attn_launches(1, 8, 1, 64, 4, 64, 148) == 1     # 4 tiles: one split of >= 4


def test_mlp_width_realises_activated_fraction():
    from paper_2504_19516_b200.device.layer import mlp_width
    from paper_2504_19516_b200.workload import MODEL_PRESETS, ModelSpec

    assert mlp_width(MODEL_PRESETS["llama3-8b"]) == 14336
    assert mlp_width(MODEL_PRESETS["moe-a22b"]) == 1280  # 0.1 x 12288, rounded to the 128-row tile
    assert mlp_width(ModelSpec("m", 1, 4096, 32, 8, 128, 14336, activated_fraction=0.5)) == 7168
    assert mlp_width(ModelSpec("m", 1, 4096, 32, 8, 128, 1024, activated_fraction=0.01)) == 128


def test_header_is_plain_c_and_cxx(tmp_path):
    """include/hp.h is the drop-in boundary: it must compile as C99 (a cgo /
    ctypes consumer) and as C++17, with no torch or CUDA types."""
    import shutil
    import subprocess
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    src = tmp_path / "use_hp.c"
    src.write_text('#include "hp.h"\nint main(void) { return hp_abi_version() == HP_ABI_VERSION ? 0 : 1; }\n')
    for cc, args in (("gcc", ["-std=c99"]), ("g++", ["-std=c++17", "-x", "c++"])):
        if shutil.which(cc) is None:
            continue
        r = subprocess.run([cc, *args, "-fsyntax-only", "-Wall", "-Werror", f"-I{root / 'include'}", str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    code = [ln for ln in (root / "include" / "hp.h").read_text().splitlines()
            if ln.strip() and not ln.strip().startswith(("/*", "*", "//"))]
    assert not any("torch" in ln or "#include <cuda" in ln for ln in code)
