"""The 2:4 compressed format and its kernels (drop-in for the reference's
pkg/src/srelu24/sparse24.py, hot-path subset).

Storage is the tensor-core layout: kept values as bf16, K-major along the
grouped axis (token-wise [rows_pad128, cols/2]; feature-wise [cols_pad128,
rows/2], i.e. the transposed operand the weight-gradient GEMM reads), plus
the tcgen05.mma.sp operand-E metadata ("hw" layout, csrc/meta.cuh) whenever
the grouped axis is a multiple of 128. The reference's views -- values and
meta as [rows, cols/4, 2] (token) or [rows/4, cols, 2] (feature) -- are
exposed as properties computed on demand on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib
from ._tensors import BF16, F32, as_matrix, dtype_code, pad128, ptr, stream
from .errors import DimensionError, MaskError, OrientationError

TOKEN_WISE = "token"
FEATURE_WISE = "feature"


class SparsifyStats:
    """Drop counts of one sparsification (ref sparse24.py:50-69). Backed by a
    device counter pair (nonzeros before, after), or a callable producing it;
    fields materialise on first access, so producing stats never forces a host
    sync."""

    __slots__ = ("total_entries", "_dev", "_host")

    def __init__(self, total_entries: int, dev_counts: torch.Tensor):
        self.total_entries = int(total_entries)
        self._dev = dev_counts
        self._host = None

    def _vals(self):
        if self._host is None:
            dev = self._dev() if callable(self._dev) else self._dev
            b, a = (int(v) for v in dev.tolist())
            self._host = (b, a)
        return self._host

    @property
    def nonzeros_before(self) -> int:
        return self._vals()[0]

    @property
    def nonzeros_after(self) -> int:
        return self._vals()[1]

    @property
    def dropped(self) -> int:
        b, a = self._vals()
        return b - a

    @property
    def sparsity_before(self) -> float:
        return 1.0 - self.nonzeros_before / self.total_entries if self.total_entries else 0.0

    @property
    def dropped_fraction_of_nonzeros(self) -> float:
        b = self.nonzeros_before
        return self.dropped / b if b else 0.0

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("total_entries", "nonzeros_before", "nonzeros_after", "dropped",
                                               "sparsity_before", "dropped_fraction_of_nonzeros")}

    def __repr__(self):
        return f"SparsifyStats({self.as_dict()})"


def _new_stats_counter(device) -> torch.Tensor:
    return torch.zeros(2, dtype=torch.int64, device=device)


@dataclass(frozen=True)
class Sparse24Matrix:
    """Packed kept values plus 2-bit in-group positions (ref sparse24.py:30-47).

    data    : bf16 kept values, K-major along the grouped axis (see module doc)
    meta_hw : uint8 tcgen05 operand-E metadata, or None when the grouped axis
              is not a multiple of 128
    """

    rows: int
    cols: int
    orientation: str
    data: torch.Tensor
    meta_hw: torch.Tensor | None = None
    meta_ref_cache: torch.Tensor | None = field(default=None, repr=False)

    @property
    def group_count(self) -> int:
        return self.rows * self.cols // 4

    @property
    def grouped_len(self) -> int:
        return self.cols if self.orientation == TOKEN_WISE else self.rows

    @property
    def values(self) -> torch.Tensor:
        """Reference layout view: [rows, cols/4, 2] (token) or [rows/4, cols, 2] (feature)."""
        if self.orientation == TOKEN_WISE:
            return self.data[: self.rows].view(self.rows, self.cols // 4, 2)
        return self.data[: self.cols].view(self.cols, self.rows // 4, 2).permute(1, 0, 2)

    @property
    def meta(self) -> torch.Tensor:
        """Reference layout uint8 positions, same shape as `values`."""
        if self.meta_ref_cache is not None:
            return self.meta_ref_cache
        if self.orientation == TOKEN_WISE:
            ref = torch.empty(self.rows, self.cols // 4, 2, dtype=torch.uint8, device=self.data.device)
            _lib.call("s24_meta_hw_to_ref", ptr(self.meta_hw), self.rows, self.cols, ptr(ref), stream())
            out = ref
        else:
            # hw metadata of the transposed operand: rows' = cols (features), K = rows
            rp = pad128(self.cols)
            ref = torch.empty(rp, self.rows // 4, 2, dtype=torch.uint8, device=self.data.device)
            _lib.call("s24_meta_hw_to_ref", ptr(self.meta_hw), rp, self.rows, ptr(ref), stream())
            out = ref[: self.cols].permute(1, 0, 2).contiguous()
        object.__setattr__(self, "meta_ref_cache", out)
        return out


def _alloc_token(rows: int, cols: int, device, with_hw: bool):
    rp = pad128(rows)
    data = torch.empty(rp, cols // 2, dtype=BF16, device=device)
    if rp > rows:
        data[rows:].zero_()
    hw = None
    if with_hw:
        hw = torch.empty(_lib.meta_hw_bytes(rows, cols), dtype=torch.uint8, device=device)
        if rp > rows:  # padding rows: valid (0,1) selectors, zero values
            hw[(rows // 128) * (cols // 128) * 2048:].fill_(0x44)
    return data, hw


def sparsify_token_wise(a):
    """Top-2-per-group along each row (ref sparse24.py:80-93).
    Returns (Sparse24Matrix, mask [rows, cols] bool, SparsifyStats)."""
    a = as_matrix(a, "a")
    rows, cols = a.shape
    if cols % 4 != 0:
        raise DimensionError(f"token-wise groups need cols % 4 == 0, got {cols}")
    with_hw = cols % 128 == 0
    data, hw = _alloc_token(rows, cols, a.device, with_hw)
    meta_ref = torch.empty(rows, cols // 4, 2, dtype=torch.uint8, device=a.device)
    mask = torch.empty(rows, cols, dtype=torch.uint8, device=a.device)
    cnt = _new_stats_counter(a.device)
    _lib.call("s24_sparsify_token", ptr(a), dtype_code(a), rows, cols, a.stride(0), ptr(data), ptr(meta_ref), ptr(hw),
              ptr(mask), ptr(cnt), stream())
    s = Sparse24Matrix(rows, cols, TOKEN_WISE, data, hw, meta_ref)
    return s, mask.bool(), SparsifyStats(rows * cols, cnt)


def sparsify_feature_wise(a):
    """Top-2-per-group down each column (ref sparse24.py:96-115)."""
    return _sparsify_feature(a, None)


def _sparsify_feature(a, fwd_mask):
    a = as_matrix(a, "a")
    rows, cols = a.shape
    m8 = None
    if fwd_mask is not None:
        m8 = _as_mask(fwd_mask, a.shape, a.device).to(torch.uint8).contiguous()
    if rows % 4 != 0:
        raise DimensionError(f"feature-wise groups need rows % 4 == 0, got {rows}")
    with_hw = rows % 128 == 0
    cp = pad128(cols)
    data = torch.zeros(cp, rows // 2, dtype=BF16, device=a.device)
    hw = None
    if with_hw:
        hw = torch.full((_lib.meta_hw_bytes(cols, rows),), 0x44, dtype=torch.uint8, device=a.device)
    meta_ref = torch.empty(rows // 4, cols, 2, dtype=torch.uint8, device=a.device)
    mask = torch.empty(rows, cols, dtype=torch.uint8, device=a.device)
    cnt = _new_stats_counter(a.device)
    _lib.call("s24_sparsify_feature_masked", ptr(a), dtype_code(a), rows, cols, a.stride(0), ptr(m8), ptr(data),
              ptr(meta_ref), ptr(hw), ptr(mask), ptr(cnt), stream())
    s = Sparse24Matrix(rows, cols, FEATURE_WISE, data, hw, meta_ref)
    return s, mask.bool(), SparsifyStats(rows * cols, cnt)


def _as_mask(mask, shape, device) -> torch.Tensor:
    if not isinstance(mask, torch.Tensor):
        mask = torch.as_tensor(mask)
    if tuple(mask.shape) != tuple(shape):
        raise DimensionError(f"mask shape {tuple(mask.shape)} does not match matrix {tuple(shape)}")
    return mask.to(device=device)


def apply_mask(a, mask) -> torch.Tensor:
    """Zero entries outside mask (ref sparse24.py:132-135)."""
    a = as_matrix(a, "a")
    m = _as_mask(mask, a.shape, a.device)
    return torch.where(m.bool(), a, torch.zeros((), dtype=a.dtype, device=a.device))


def sparsify_feature_wise_masked(a, fwd_mask):
    """Zero entries outside fwd_mask, then sparsify feature-wise; masked-out
    values do not count as dropped (ref sparse24.py:118-129). One device pass:
    the mask is applied while the kernel reads the operand."""
    return _sparsify_feature(a, fwd_mask)


def compress_token_wise_with_mask(a, mask) -> Sparse24Matrix:
    """Exact token-wise compression on a given 2-of-4 mask (ref
    sparse24.py:138-154). Raises MaskError unless every group has exactly 2
    mask bits (checked on the device, one host sync)."""
    a = as_matrix(a, "a")
    rows, cols = a.shape
    m = _as_mask(mask, a.shape, a.device)
    if cols % 4 != 0:
        raise DimensionError(f"mask/matrix shapes unusable: {tuple(m.shape)} vs {tuple(a.shape)}")
    m8 = m.to(torch.uint8).contiguous()
    with_hw = cols % 128 == 0
    data, hw = _alloc_token(rows, cols, a.device, with_hw)
    meta_ref = torch.empty(rows, cols // 4, 2, dtype=torch.uint8, device=a.device)
    bad = torch.zeros(1, dtype=torch.int32, device=a.device)
    _lib.call("s24_compress_token_with_mask", ptr(a), dtype_code(a), rows, cols, a.stride(0), ptr(m8), ptr(data),
              ptr(meta_ref), ptr(hw), ptr(bad), stream())
    if int(bad.item()):
        raise MaskError("mask must set exactly 2 bits per group of 4")
    return Sparse24Matrix(rows, cols, TOKEN_WISE, data, hw, meta_ref)


def decompress(s: Sparse24Matrix, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """Dense matrix with kept values at their positions (ref sparse24.py:157-167)."""
    out = torch.empty(s.rows, s.cols, dtype=out_dtype, device=s.data.device)
    code = _lib.F32 if out_dtype == F32 else _lib.BF16
    if s.orientation == TOKEN_WISE:
        use_hw = s.meta_hw is not None
        _lib.call("s24_decompress_token", ptr(s.data), None if use_hw else ptr(s.meta), ptr(s.meta_hw) if use_hw else None,
                  s.rows, s.cols, ptr(out), code, s.cols, stream())
    else:
        use_hw = s.meta_hw is not None
        _lib.call("s24_decompress_feature", ptr(s.data), None if use_hw else ptr(s.meta),
                  ptr(s.meta_hw) if use_hw else None, s.rows, s.cols, ptr(out), code, s.cols, stream())
    return out


def _hw_operand(s: Sparse24Matrix):
    """(values, hw meta) of a compressed matrix as the sparse GEMM's A operand;
    re-pads the grouped axis to a multiple of 128 when needed."""
    if s.meta_hw is not None:
        return s.data, s.meta_hw, s.grouped_len
    # grouped axis not a multiple of 128: rebuild a padded operand on the device
    dense = decompress(s, BF16)
    if s.orientation == FEATURE_WISE:
        dense = dense.t().contiguous()
    m, k = dense.shape
    kp = pad128(k)
    padded = torch.zeros(m, kp, dtype=BF16, device=dense.device)
    padded[:, :k] = dense
    t, _, _ = sparsify_token_wise(padded)  # exact: every group already has <= 2 nonzeros
    return t.data, t.meta_hw, kp


def _spmm(vals, meta_hw, m: int, k: int, b: torch.Tensor, out_dtype) -> torch.Tensor:
    kb, n = b.shape
    kpad = vals.shape[1] * 2
    if kpad != k:
        bp = torch.zeros(kpad, n, dtype=BF16, device=b.device)
        bp[:k] = b
        b = bp
    npad = (n + 31) // 32 * 32
    if npad != n:
        bp = torch.zeros(b.shape[0], npad, dtype=BF16, device=b.device)
        bp[:, :n] = b
        b = bp
    out = torch.empty(m, npad, dtype=out_dtype, device=b.device)
    code = _lib.F32 if out_dtype == F32 else _lib.BF16
    _lib.call("s24_spmm", ptr(vals), ptr(meta_hw), ptr(b), 1, npad, m, npad, kpad, ptr(out), code, npad, None, 0, -1, None, 0,
              stream())
    return out[:, :n] if npad != n else out


def sp_gemm(s: Sparse24Matrix, b, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """Token-wise 2:4 A times dense B on tcgen05.mma.sp (ref sparse24.py:170-192)."""
    if s.orientation != TOKEN_WISE:
        raise OrientationError("sp_gemm needs a token-wise operand")
    b = as_matrix(b, "b", BF16)
    if s.cols != b.shape[0]:
        raise DimensionError(f"inner dimensions differ: {s.rows}x{s.cols} x {tuple(b.shape)}")
    vals, hw, _ = _hw_operand(s)
    return _spmm(vals, hw, s.rows, s.cols, b, out_dtype)


def sp_gemm_t(s: Sparse24Matrix, b, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """Feature-wise 2:4 A as A^T @ B, reduction over tokens (ref sparse24.py:195-216).
    The feature-wise storage is already the K-major sparse operand."""
    if s.orientation != FEATURE_WISE:
        raise OrientationError("sp_gemm_t needs a feature-wise operand")
    b = as_matrix(b, "b", BF16)
    if s.rows != b.shape[0]:
        raise DimensionError(f"reduction dimensions differ: {s.rows}x{s.cols} x {tuple(b.shape)}")
    vals, hw, _ = _hw_operand(s)
    return _spmm(vals, hw, s.cols, s.rows, b, out_dtype)


def sp_gemm_macs(rows: int, cols: int, n: int) -> int:
    """MACs of either sparse kernel: half the dense count (ref sparse24.py:219-221)."""
    return rows * cols * n // 2
