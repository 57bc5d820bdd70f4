"""Split GEMM (paper Optimization 1; drop-in for the reference's
pkg/src/srelu24/splitgemm.py).

Features are ranked by nonzero count; the ceil(ratio*h) sparsest go through a
feature-wise 2:4 sparse GEMM, the rest through an exact dense GEMM, and both
partial products scatter into the output by feature index inside the GEMM
epilogue (row map). The plan is computed on the device (K7) from counts that
the forward GEMM's epilogue already produced, so no host sync is needed: its
sizes follow from h and the ratio alone.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from ._tensors import BF16, F32, as_matrix, pad128, ptr, stream
from .errors import ConfigError, DimensionError
from .sparse24 import (
    SparsifyStats,
    TOKEN_WISE,
    apply_mask,
    sp_gemm_macs,
    sparsify_feature_wise,
)
from .matcore import gemm_macs


@dataclass(frozen=True)
class SplitPlan:
    """Partition of feature indices (ref splitgemm.py:17-25). Index lists are
    int32 device tensors; feat_pos[j] = rank of j in the sparse list, or
    -(rank in the dense list) - 1."""

    hidden_dim: int
    ratio: float
    counts: torch.Tensor
    sparse_features: torch.Tensor
    dense_features: torch.Tensor
    feat_pos: torch.Tensor

    @property
    def n_sparse(self) -> int:
        return int(self.sparse_features.shape[0])

    @property
    def n_dense(self) -> int:
        return int(self.dense_features.shape[0])

    @cached_property
    def paired_row_map(self) -> torch.Tensor:
        """Output row of each row of a paired-layout operand: dense feature r
        twice (rows 2r, 2r+1), then the sparse features."""
        return torch.cat([self.dense_features.repeat_interleave(2), self.sparse_features]).to(torch.int32)


def column_nonzero_counts(a) -> torch.Tensor:
    """counts[j] = number of nonzero entries in column j (ref splitgemm.py:28-30).
    (On the FFN hot path these counts come out of the K1 epilogue instead.)"""
    a = as_matrix(a, "a")
    return (a != 0).sum(dim=0).to(torch.int64)


def ceil_fraction(ratio: float, h: int) -> int:
    """ceil(ratio*h), exact for integral products (ref splitgemm.py:33-38)."""
    x = ratio * h
    if abs(x - round(x)) < 1e-9:
        return int(round(x))
    return math.ceil(x)


def partition_features(counts, ratio: float, launch_stream=None) -> SplitPlan:
    """Stable ascending (count, index) order; the first ceil(ratio*h) features
    are sparse, both lists ascending (ref splitgemm.py:41-52). Runs on the
    device (radix select + block scan, csrc/sparse_capi.cu k_plan).
    launch_stream: run the kernel there (outputs are still allocated on the
    current stream, which must wait for launch_stream before reading them)."""
    if not 0.0 <= ratio <= 1.0:
        raise ConfigError(f"split ratio must be in [0, 1], got {ratio}")
    if isinstance(counts, np.ndarray) or not isinstance(counts, torch.Tensor):
        counts = torch.as_tensor(np.asarray(counts, dtype=np.int64))
    if not counts.is_cuda:
        counts = counts.cuda()
    h = int(counts.shape[0])
    c32 = counts.to(torch.int32).contiguous()
    k = ceil_fraction(ratio, h)
    dev = c32.device
    sp = torch.empty(max(k, 0), dtype=torch.int32, device=dev)
    de = torch.empty(max(h - k, 0), dtype=torch.int32, device=dev)
    pos = torch.empty(h, dtype=torch.int32, device=dev)
    if h:
        sp_buf = sp if k else torch.empty(1, dtype=torch.int32, device=dev)
        de_buf = de if h - k else torch.empty(1, dtype=torch.int32, device=dev)
        st = launch_stream.cuda_stream if launch_stream is not None else stream()
        _lib.call("s24_plan", ptr(c32), h, k, ptr(sp_buf), ptr(de_buf), ptr(pos), st)
    return SplitPlan(h, ratio, counts, sp, de, pos)


def pad_plan(plan: SplitPlan, h_pad: int, launch_stream=None) -> SplitPlan:
    """The plan of h features extended to h_pad >= h features: the padding
    features [h, h_pad) (all-zero columns of a padded FFN) become extra sparse
    ranks after the real ones; dense features are unchanged."""
    h = plan.hidden_dim
    if h_pad == h:
        return plan
    dev, ns, extra = plan.feat_pos.device, plan.n_sparse, h_pad - h
    # outputs allocated on the current stream (the consumer's), filled on launch_stream
    sp = torch.empty(ns + extra, dtype=torch.int32, device=dev)
    pos = torch.empty(h_pad, dtype=torch.int32, device=dev)
    counts = torch.empty(h_pad, dtype=plan.counts.dtype, device=dev)
    with torch.cuda.stream(launch_stream or torch.cuda.current_stream(dev)):
        sp[:ns].copy_(plan.sparse_features)
        sp[ns:].copy_(torch.arange(h, h_pad, dtype=torch.int32, device=dev))
        pos[:h].copy_(plan.feat_pos)
        pos[h:].copy_(torch.arange(ns, ns + extra, dtype=torch.int32, device=dev))
        counts[:h].copy_(plan.counts)
        counts[h:].zero_()
    return SplitPlan(h_pad, plan.ratio, counts, sp, plan.dense_features, pos)


def partition_features_padded(counts, ratio: float, h_valid: int, launch_stream=None):
    """partition_features over the first h_valid features of a padded FFN
    (the reference's plan, returned first) and its padded device form."""
    if h_valid == counts.shape[0]:
        plan = partition_features(counts, ratio, launch_stream)
        return plan, plan
    plan = partition_features(counts[:h_valid], ratio, launch_stream)
    return plan, pad_plan(plan, counts.shape[0], launch_stream)


def split_gemm_macs(n: int, d: int, plan: SplitPlan) -> int:
    """Exact MAC count n*d*(|sparse|/2 + |dense|) (ref splitgemm.py:84-88)."""
    return sp_gemm_macs(n, plan.n_sparse, d) + gemm_macs(plan.n_dense, n, d)


@dataclass
class FeatureSplit:
    """Device operand of one split weight-gradient GEMM, produced by K4 in the
    paired layout (csrc/k4.cuh): vs rows [0, pair_rows) hold the dense
    features as fixed-selector 2:4 row pairs (rows 2r, 2r+1 = tokens 4j, 4j+1
    and 4j+2, 4j+3 of dense rank r), sparse rank s is row pair_rows + s."""

    vs: torch.Tensor  # bf16 [pad128(pair_rows + n_sparse), n/2] feature-wise 2:4 values, K-major along tokens
    es: torch.Tensor  # hw metadata, rows = operand rows, K = tokens
    stats: SparsifyStats
    pair_rows: int

    def rows(self, plan: "SplitPlan") -> int:
        """Rows of the 2:4 operand vs that carry features."""
        return self.pair_rows + plan.n_sparse


def feature_split(vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan,
                  with_stats: bool = False, nonneg: bool = False) -> FeatureSplit:
    """K4: token-wise compressed [n, h] (vals + hw meta, n and h multiples of
    128) -> the paired-layout feature-wise split (the apply_mask / gather /
    sparsify_feature_wise part of ref splitgemm.py:72-80, without a dense
    round trip). with_stats counts the sparse features' nonzeros before /
    after on the device (the reference computes and discards them,
    splitgemm.py:75). nonneg=True declares the values >= 0 (the relu^2
    activation), letting K4 rank raw values."""
    fs = alloc_feature_split(vals, meta_hw, n, h, plan)
    ns, nd = plan.n_sparse, plan.n_dense
    if with_stats:
        cnt = torch.zeros(2, dtype=torch.int64, device=vals.device)
        _lib.call("s24_feature_split", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), ns, nd, ptr(fs.vs),
                  ptr(fs.es), None, ptr(cnt), int(nonneg), fs.pair_rows, stream())
        fs.stats = SparsifyStats(n * ns, cnt)
    else:
        run_feature_split(fs, vals, meta_hw, n, h, plan, nonneg=nonneg)
    return fs


def alloc_feature_split(vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan) -> FeatureSplit:
    """Output buffers of one K4 job (filled by run_feature_split). Its drop
    statistics are not counted on the hot path -- the reference discards them
    (splitgemm.py:75) -- and are recounted on the device only if someone reads
    them."""
    dev = vals.device
    ns, nd = plan.n_sparse, plan.n_dense

    def recount():
        return feature_split(vals, meta_hw, n, h, plan, with_stats=True).stats._dev

    rows = ns + 2 * nd
    vs = torch.empty(max(pad128(rows), 128), n // 2, dtype=BF16, device=dev)
    es = torch.empty(_lib.meta_hw_bytes(max(rows, 1), n), dtype=torch.uint8, device=dev)
    return FeatureSplit(vs, es, SparsifyStats(n * ns, recount), 2 * nd)


def run_feature_split(fs: FeatureSplit, vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int,
                      plan: SplitPlan, nonneg: bool = False, nan_flag: torch.Tensor | None = None) -> None:
    """Fill preallocated K4 outputs on the current stream (no drop counting).
    nan_flag: K1's "a kept value is NaN" word; with nonneg it switches K4 back
    to NaN-aware ranking."""
    _lib.call("s24_feature_split_x", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), plan.n_sparse,
              plan.n_dense, ptr(fs.vs), ptr(fs.es), int(nonneg), ptr(nan_flag), stream())


def side_stream(device, which: int = 0) -> torch.cuda.Stream:
    """Per-device streams that carry K4 and the permuted copies next to the
    main-stream GEMMs (0: the forward's, 1: the backward's; the e4m3 path also
    quantizes the weight gradients' B operands on 2: x_in^T, 3: g_c^T)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    st = _side_streams.get((idx, which))
    if st is None:
        st = _side_streams[(idx, which)] = torch.cuda.Stream(device=device)
    return st


_side_streams: dict[tuple[int, int], torch.cuda.Stream] = {}


def split_weight_grad(fs: FeatureSplit, plan: SplitPlan, b: torch.Tensor, n: int, out: torch.Tensor,
                      transposed: bool) -> None:
    """out[S] = sparse(fs)^T b and out[D] = dense(fs)^T b in ONE 2:4 GEMM over
    the paired-layout operand (the dense features' row pairs are summed in the
    epilogue), rows scattered by feature index. b: bf16 [n, d] (K = tokens,
    MN-major). transposed=True writes out as [d, h] (dW1 layout)."""
    d = b.shape[1]
    rows = fs.rows(plan)
    if rows:
        code = _lib.F32 if out.dtype == F32 else _lib.BF16
        _lib.call("s24_spmm", ptr(fs.vs), ptr(fs.es), ptr(b), 1, b.stride(0), rows, d, n, ptr(out), code,
                  out.shape[1], ptr(plan.paired_row_map), int(transposed), rows, None, fs.pair_rows, stream())


def split_weight_grad_pair(fa: FeatureSplit, fb: FeatureSplit, plan: SplitPlan, b_a: torch.Tensor,
                           b_b: torch.Tensor, n: int, out_a: torch.Tensor, out_b: torch.Tensor) -> None:
    """split_weight_grad for two operands sharing one plan and one (rows, d, n)
    shape: out_a = split(fa)^T b_a (row-major [h, d]) and out_b =
    (split(fb)^T b_b)^T (transposed [d, h]) in ONE grouped 2:4 launch."""
    d = b_a.shape[1]
    if b_b.shape[1] != d or out_a.dtype != out_b.dtype:
        raise DimensionError("paired weight gradients need equal widths and output dtypes")
    if fa.pair_rows != fb.pair_rows:
        raise DimensionError("both operands must come from the same plan")
    rows = fa.rows(plan)
    if not rows:
        return
    code = _lib.F32 if out_a.dtype == F32 else _lib.BF16
    rm = ptr(plan.paired_row_map)
    _lib.call("s24_spmm_pair", 1, rows, d, n, code,
              ptr(fa.vs), ptr(fa.es), ptr(b_a), b_a.stride(0), ptr(out_a), out_a.shape[1], rm, 0, None,
              ptr(fb.vs), ptr(fb.es), ptr(b_b), b_b.stride(0), ptr(out_b), out_b.shape[1], rm, 1, None,
              fa.pair_rows, stream())


def split_gemm_t(a, fwd_mask, b, plan: SplitPlan, out_dtype: torch.dtype = F32) -> torch.Tensor:
    """Masked a^T b via one feature-wise 2:4 GEMM plus one dense GEMM, rows
    scattered by feature index (ref splitgemm.py:55-81). Generic entry point
    for arbitrary (mask, a); the FFN hot path calls feature_split +
    split_weight_grad on the already-compressed activation instead."""
    a = as_matrix(a, "a")
    n, h = a.shape
    if n % 4 != 0:
        raise DimensionError(f"feature-wise groups need rows % 4 == 0, got {n}")
    if plan.hidden_dim != h:
        raise DimensionError(f"plan built for {plan.hidden_dim} features, matrix has {h}")
    b = as_matrix(b, "b", BF16)
    if b.shape[0] != n:
        raise DimensionError(f"reduction dimensions differ: {tuple(a.shape)} x {tuple(b.shape)}")
    am = apply_mask(a, fwd_mask)
    d = b.shape[1]
    out = torch.zeros(h, d, dtype=out_dtype, device=a.device)
    if n % 128 == 0 and h % 128 == 0 and d % 32 == 0:
        from .sparse24 import sparsify_token_wise

        # exact token-wise compression of the masked operand keeps every value
        # whose group has <= 2 nonzeros; for general masks fall back to the
        # per-partition path below
        if bool(((am.view(n, h // 4, 4) != 0).sum(-1) <= 2).all()):
            t, _, _ = sparsify_token_wise(am)
            fs = feature_split(t.data, t.meta_hw, n, h, plan)
            split_weight_grad(fs, plan, b, n, out, transposed=False)
            return out
    from .sparse24 import sp_gemm_t
    from .matcore import gemm_at

    if plan.n_sparse:
        sidx = plan.sparse_features.long()
        s, _, _ = sparsify_feature_wise(am[:, sidx].contiguous())
        out[sidx] = sp_gemm_t(s, b, out_dtype)
    if plan.n_dense:
        didx = plan.dense_features.long()
        out[didx] = gemm_at(am[:, didx].contiguous(), b, out_dtype)
    return out
