"""Dense GEMMs and token permutations of the drop-in API.

Mirrors the hot-path subset of the reference's pkg/src/srelu24/matcore.py:
`gemm` / `gemm_at` (:71-106) run on the tcgen05 GEMM with fp32 accumulation
(tolerance-level, not ascending-order, agreement with the reference), and the
seeded permutation helpers (:269-307) keep the reference's exact semantics:
the permutation itself is drawn on the host by the same PCG64 Fisher-Yates
stream (so it is bit-identical), then cached on the device.
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _lib
from ._tensors import BF16, F32, as_matrix, ptr, stream
from .errors import DimensionError, PrecisionError

WORKING = np.float32
ORACLE = np.float64


def gemm_macs(m: int, k: int, n: int) -> int:
    """Multiply-accumulate count of a dense m x k x n product (ref matcore.py:109-111)."""
    return m * k * n


def _out_code(dtype: torch.dtype) -> int:
    if dtype == F32:
        return _lib.F32
    if dtype == BF16:
        return _lib.BF16
    raise PrecisionError(f"unsupported output dtype {dtype}")


def gemm(a, b, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """c = a @ b on tensor cores (bf16 operands, fp32 accumulation).
    Drop-in for ref matcore.py:71-87."""
    a = as_matrix(a, "a", BF16)
    b = as_matrix(b, "b", BF16)
    m, k = a.shape
    kb, n = b.shape
    if kb != k:
        raise DimensionError(f"inner dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    out = torch.empty(m, n, device=a.device, dtype=out_dtype)
    if n % 32:
        # the tcgen05 epilogue stores 32-column chunks; pad N
        npad = (n + 31) // 32 * 32
        bp = torch.zeros(k, npad, device=a.device, dtype=BF16)
        bp[:, :n] = b
        return gemm(a, bp, out_dtype)[:, :n].contiguous()
    _lib.call("s24_gemm", ptr(a), 0, k, ptr(b), 1, n, m, n, k, ptr(out), _out_code(out_dtype), n, None, 0, -1, None,
              stream())
    return out


def gemm_at(a, b, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """c = a^T @ b without materialising the transpose (A read MN-major).
    Drop-in for ref matcore.py:90-106."""
    a = as_matrix(a, "a", BF16)
    b = as_matrix(b, "b", BF16)
    k, m = a.shape
    kb, n = b.shape
    if kb != k:
        raise DimensionError(f"reduction dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    if n % 32 or m % 8:
        npad, mpad = (n + 31) // 32 * 32, (m + 7) // 8 * 8
        ap = torch.zeros(k, mpad, device=a.device, dtype=BF16)
        ap[:, :m] = a
        bp = torch.zeros(k, npad, device=a.device, dtype=BF16)
        bp[:, :n] = b
        return gemm_at(ap, bp, out_dtype)[:m, :n].contiguous()
    out = torch.empty(m, n, device=a.device, dtype=out_dtype)
    _lib.call("s24_gemm", ptr(a), 1, m, ptr(b), 1, n, m, n, k, ptr(out), _out_code(out_dtype), n, None, 0, -1, None,
              stream())
    return out


# ---------------------------------------------------------------- permutations

_CACHE_ENTRIES = 16  # permutations kept per cache (LRU): distinct token counts are few in practice
_perm_cache: "OrderedDict[tuple[int, int], np.ndarray]" = OrderedDict()
_dev_cache: "OrderedDict[tuple[int, int, int], tuple[torch.Tensor, torch.Tensor]]" = OrderedDict()
_cache_lock = threading.Lock()


def _lru_get(cache: OrderedDict, key):
    with _cache_lock:
        hit = cache.get(key)
        if hit is not None:
            cache.move_to_end(key)
        return hit


def _lru_put(cache: OrderedDict, key, value) -> None:
    with _cache_lock:
        cache[key] = value
        cache.move_to_end(key)
        while len(cache) > _CACHE_ENTRIES:
            cache.popitem(last=False)


def make_permutation(seed: int, n: int) -> np.ndarray:
    """Fisher-Yates shuffle of [0, n) driven by numpy's PCG64(seed), swapping
    from the top with j = integers(0, i + 1) (ref matcore.py:269-280). Same
    (seed, n) -> same permutation on every platform; LRU-cached per (seed, n)."""
    key = (int(seed), int(n))
    hit = _lru_get(_perm_cache, key)
    if hit is not None:
        return hit.copy()
    gen = np.random.Generator(np.random.PCG64(seed))
    perm = np.arange(n, dtype=np.int64)
    draw = gen.integers
    for i in range(n - 1, 0, -1):
        j = int(draw(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    _lru_put(_perm_cache, key, perm)
    return perm.copy()


def device_permutation(seed: int, n: int, device=None) -> tuple[torch.Tensor, torch.Tensor]:
    """(perm, inverse) as int32 device tensors, LRU-cached per (seed, n, device)."""
    dev = torch.device(device or "cuda")
    di = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (int(seed), int(n), di)
    hit = _lru_get(_dev_cache, key)
    if hit is None:
        p = make_permutation(seed, n)
        inv = np.empty_like(p)
        inv[p] = np.arange(n)
        hit = (torch.from_numpy(p.astype(np.int32)).to(dev), torch.from_numpy(inv.astype(np.int32)).to(dev))
        _lru_put(_dev_cache, key, hit)
    return hit


def _as_index(p, n: int, device) -> torch.Tensor:
    if isinstance(p, np.ndarray):
        if p.ndim != 1 or len(p) != n:
            raise DimensionError(f"permutation of size {p.shape} cannot act on {n} rows")
        return torch.from_numpy(p.astype(np.int32)).to(device)
    if p.dim() != 1 or p.shape[0] != n:
        raise DimensionError(f"permutation of size {tuple(p.shape)} cannot act on {n} rows")
    return p.to(device=device, dtype=torch.int32)


def gather_rows(a: torch.Tensor, src: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = a[src[i]] on the device (K6). out may have more (padding) rows."""
    n = src.shape[0]
    if out is None:
        out = torch.empty(n, a.shape[1], device=a.device, dtype=a.dtype)
    rb = a.shape[1] * a.element_size()
    _lib.call("s24_gather_rows", ptr(a), n, rb, a.stride(0) * a.element_size(), ptr(src), ptr(out),
              out.stride(0) * out.element_size(), stream())
    return out


def permute_rows(a, p) -> torch.Tensor:
    """out[p[i], :] = a[i, :] (ref matcore.py:291-296)."""
    a = as_matrix(a, "a")
    pi = _as_index(p, a.shape[0], a.device)
    inv = torch.empty_like(pi)
    inv[pi.long()] = torch.arange(a.shape[0], device=a.device, dtype=torch.int32)
    return gather_rows(a, inv)


def inverse_permute_rows(a, p) -> torch.Tensor:
    """out[i, :] = a[p[i], :] (ref matcore.py:299-302)."""
    a = as_matrix(a, "a")
    return gather_rows(a, _as_index(p, a.shape[0], a.device))


def compose_permutations(q, p):
    """Permutation equivalent to applying p first, then q (ref matcore.py:305-307)."""
    return q[p]
