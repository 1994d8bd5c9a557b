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
