"""The C-ABI library loads without a GPU and exports every entry point that
include/s24.h declares (no compute calls here)."""

import re
from pathlib import Path

import pytest

from paper_2503_16672_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "s24.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(s24_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not _lib.LIB_PATH.exists():
        from paper_2503_16672_b200.build import build

        build()
    return _lib.load()


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for must in ("s24_sparsify_token", "s24_sparsify_feature", "s24_spmm", "s24_gemm", "s24_fwd_gemm1_fused",
                 "s24_bwd_dact_fused", "s24_feature_split", "s24_plan", "s24_gather_rows", "s24_last_error"):
        assert must in syms


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_every_bound_symbol_is_declared():
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_host_only_helpers(lib):
    assert "sm_100a" in _lib.version()
    assert _lib.meta_hw_bytes(4096, 2048) == 4096 * 2048 // 8
    assert _lib.meta_hw_bytes(200, 256) == 256 * 256 // 8


def test_argument_validation_needs_no_device(lib):
    # shape errors are detected on the host before any launch
    with pytest.raises(Exception) as e:
        _lib.call("s24_sparsify_token", None, 0, 4, 6, 6, None, None, None, None, None, None)
    assert type(e.value).__name__ == "DimensionError"
    with pytest.raises(Exception) as e:
        _lib.call("s24_plan", None, 10, 11, None, None, None, None)
    assert type(e.value).__name__ == "ConfigError"
    with pytest.raises(Exception) as e:
        _lib.call("s24_spmm", None, None, None, 1, 64, 128, 64, 100, None, 0, 64, None, 0, -1, None, 0, None)
    assert type(e.value).__name__ == "DimensionError"
