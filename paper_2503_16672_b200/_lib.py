"""ctypes binding of libs24.so (the C ABI declared in include/s24.h).

This module is the only place that touches the shared library. There is no
CPU fallback: if the library is missing or no CUDA device is present, calls
raise BackendError loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from . import errors

_PKG = Path(__file__).resolve().parent
# S24_LIB: alternative build of the same library (A/B experiments, scripts/)
LIB_PATH = Path(os.environ.get("S24_LIB") or (_PKG / "libs24.so"))

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
INT = ctypes.c_int

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "s24_sparsify_token": [P, INT, I64, I64, I64, P, P, P, P, P, P],
    "s24_sparsify_feature": [P, INT, I64, I64, I64, P, P, P, P, P, P],
    "s24_sparsify_feature_masked": [P, INT, I64, I64, I64, P, P, P, P, P, P, P],
    "s24_compress_token_with_mask": [P, INT, I64, I64, I64, P, P, P, P, P, P],
    "s24_decompress_token": [P, P, P, I64, I64, P, INT, I64, P],
    "s24_decompress_feature": [P, P, P, I64, I64, P, INT, I64, P],
    "s24_meta_hw_to_ref": [P, I64, I64, P, P],
    "s24_meta_ref_to_hw": [P, I64, I64, P, P],
    "s24_gather_rows": [P, I64, I64, I64, P, P, I64, P],
    "s24_plan": [P, I64, I64, P, P, P, P],
    "s24_timestamp": [P, P],
    "s24_clock_probe": [P, INT, I64, P],
    "s24_feature_split_x": [P, P, I64, I64, P, I64, I64, P, P, INT, P, P],
    "s24_feature_split": [P, P, I64, I64, P, I64, I64, P, P, P, P, INT, I64, P],
    "s24_gemm": [P, INT, I64, P, INT, I64, I64, I64, I64, P, INT, I64, P, INT, I64, P, P],
    "s24_gemm_splitk": [P, INT, I64, P, INT, I64, I64, I64, I64, INT, P, P, INT, I64, P, INT, P],
    "s24_spmm": [P, P, P, INT, I64, I64, I64, I64, P, INT, I64, P, INT, I64, P, I64, P],
    "s24_spmm_pair": [INT, I64, I64, I64, INT, P, P, P, I64, P, I64, P, INT, P, P, P, P, I64, P, I64, P, INT, P, I64, P],
    "s24_fwd_gemm1_fused": [P, I64, P, I64, I64, I64, I64, P, P, P, P, P, P],
    "s24_bwd_dact_fused": [P, I64, P, I64, I64, I64, I64, P, P, P, P],
    "s24_gemm_relu2": [P, I64, P, I64, I64, I64, I64, P, I64, P],
    "s24_gemm_dact": [P, I64, P, I64, I64, I64, I64, P, I64, P, I64, P],
    "s24_fp8_quant_rows": [P, INT, I64, I64, I64, P, I64, P, I64, P, P, I64, P, I64, P],
    "s24_fp8_quant_cols_t": [P, INT, I64, I64, I64, P, I64, P, P, P],
    "s24_meta_hw_to_f8": [P, I64, I64, P, P],
    "s24_e4m3_encode": [P, I64, P, P],
    "s24_gemm_f8": [P, I64, P, I64, I64, I64, I64, P, P, P, INT, I64, P, INT, I64, P],
    "s24_spmm_f8": [P, P, P, I64, I64, I64, I64, P, P, P, INT, I64, P, INT, I64, P, I64, P],
    "s24_spmm_pair_f8": [I64, I64, I64, INT, P, P, P, I64, P, P, P, I64, P, INT, P, P, P, P, I64, P, P, P, I64, P, INT,
                         P, I64, P],
    "s24_fwd_gemm1_f8": [P, I64, P, I64, I64, I64, I64, P, P, P, P, P, P, P, P, P],
    "s24_bwd_dact_f8": [P, I64, P, I64, I64, I64, I64, P, P, P, P, P, P],
    "s24_last_error": [],
    "s24_version": [],
    "s24_meta_hw_bytes": [I64, I64],
}
_RESTYPES = {"s24_last_error": ctypes.c_char_p, "s24_version": ctypes.c_char_p, "s24_meta_hw_bytes": I64}

F32, BF16 = 0, 1

_CODE_TO_EXC = {
    1: errors.DimensionError,
    2: errors.OrientationError,
    3: errors.MaskError,
    4: errors.PrecisionError,
    5: errors.ConfigError,
    6: errors.StateError,
    7: errors.BackendError,
}


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raises BackendError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise errors.BackendError(
                    f"{LIB_PATH} not built; run `python -m paper_2503_16672_b200.build` "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, INT)
            _lib = lib
    return _lib


_tracer = None


def set_tracer(tracer) -> None:
    """Install (or clear with None) an object with before(name, args) / after(name)
    hooks around every entry-point call; bench.py uses it to bracket each
    kernel with CUDA events on the launching stream and to count launches."""
    global _tracer
    _tracer = tracer


def call(name: str, *args) -> None:
    """Invoke an s24_* entry point and map a non-zero status to the exception."""
    tr = _tracer
    if tr is not None:
        tr.before(name, args)
    rc = getattr(load(), name)(*args)
    if tr is not None:
        tr.after(name)
    if rc != 0:
        msg = load().s24_last_error().decode(errors="replace")
        raise _CODE_TO_EXC.get(rc, errors.BackendError)(msg)


def meta_hw_bytes(rows: int, cols: int) -> int:
    return int(load().s24_meta_hw_bytes(rows, cols))


def version() -> str:
    return load().s24_version().decode()
