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
    def identity_rows(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(row map, row_valid) of an identity-layout operand (csrc/k4id.cuh):
        dense pairs, zero padding to 128 rows, then every feature in index
        order; the dense features' and padding rows are skipped."""
        nd, h = self.n_dense, self.hidden_dim
        pad = pad128(2 * nd) - 2 * nd
        dev = self.feat_pos.device
        rmap = torch.cat([self.dense_features.repeat_interleave(2), torch.zeros(pad, dtype=torch.int32, device=dev),
                          torch.arange(h, dtype=torch.int32, device=dev)]).to(torch.int32)
        valid = torch.cat([torch.zeros(2 * nd, dtype=torch.int32, device=dev),
                           torch.full((pad,), -1, dtype=torch.int32, device=dev), self.feat_pos]).to(torch.int32)
        return rmap, valid

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
    """Device operands of one split weight-gradient GEMM, produced by K4."""

    vs: torch.Tensor  # bf16 [pad128(n_sparse), n/2] feature-wise 2:4 values, K-major along tokens
    es: torch.Tensor  # hw metadata, rows = sparse rank, K = tokens
    vd: torch.Tensor | None  # bf16 [pad128(n_dense), n] dense features, transposed (None when paired)
    stats: SparsifyStats
    # >= 0: paired layout (csrc/k4.cuh): vs rows [0, pair_rows) are the dense
    # features as fixed-selector 2:4 row pairs, sparse rank s is row pair_rows + s
    pair_rows: int = -1
    # identity layout (csrc/k4id.cuh): the dense pairs padded to 128 rows,
    # then every feature f at row pair_pad + f
    identity: bool = False

    def rows(self, plan: "SplitPlan") -> int:
        """Rows of the 2:4 operand vs that carry features."""
        if self.identity:
            return pad128(self.pair_rows) + plan.hidden_dim
        return max(self.pair_rows, 0) + plan.n_sparse

    def gemm_rows(self, plan: "SplitPlan"):
        """(M, row map, row_valid) of the split weight-gradient GEMM over vs."""
        if self.identity:
            rmap, valid = plan.identity_rows
            return self.rows(plan), rmap, valid
        return self.rows(plan), plan.paired_row_map, None


def feature_split(vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan,
                  dense_only: bool = False, with_stats: bool = False, nonneg: bool = False,
                  paired: bool = False, identity: bool = False) -> FeatureSplit:
    """K4: token-wise compressed [n, h] (vals + hw meta, n and h multiples of
    128) -> feature-wise 2:4 of the sparse features + transposed dense
    features (the apply_mask / gather / sparsify_feature_wise part of ref
    splitgemm.py:72-80, without a dense round trip). dense_only=True produces
    only the dense columns (the FFN hot path gets the sparse operand from the
    K1/K3 epilogues). nonneg=True declares the values >= 0 and NaN-free (the
    relu^2 activation), letting K4 rank raw values. paired=True writes the
    dense features into vs as fixed-selector 2:4 row pairs (one sparse GEMM
    then covers the whole split product, see split_weight_grad); identity=True
    the coalesced identity-order variant of that (csrc/k4id.cuh)."""
    fs = alloc_feature_split(vals, meta_hw, n, h, plan, dense_only, paired, identity)
    ns, nd = plan.n_sparse, plan.n_dense
    cnt = torch.zeros(2, dtype=torch.int64, device=vals.device) if with_stats else None
    if fs.identity:
        _lib.call("s24_feature_split_id", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), nd, ptr(fs.vs),
                  ptr(fs.es), ptr(cnt), int(nonneg), stream())
    else:
        _lib.call("s24_feature_split", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), ns, nd, ptr(fs.vs),
                  ptr(fs.es), ptr(fs.vd), ptr(cnt), int(nonneg), fs.pair_rows, stream())
    if with_stats:
        fs.stats = SparsifyStats(n * ns, cnt)
    return fs


def frame_rows_compressed(vals: torch.Tensor, meta_hw: torch.Tensor, row_map: torch.Tensor, n: int, h: int):
    """Token-wise compressed [n, h] (vals + hw metadata) with its rows
    gathered: row j of the result is row row_map[j] (for statistics and API
    views of token-order storage; not on the hot path)."""
    from .sparse24 import TOKEN_WISE, Sparse24Matrix

    rows = row_map[:n].long()
    ref = Sparse24Matrix(n, h, TOKEN_WISE, vals, meta_hw).meta[rows].contiguous()
    v = torch.zeros_like(vals)
    v[:n] = vals[rows]
    hw = torch.full_like(meta_hw, 0x44)
    _lib.call("s24_meta_ref_to_hw", ptr(ref), n, h, ptr(hw), stream())
    return v, hw


def alloc_feature_split(vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan,
                        dense_only: bool = False, paired: bool = False, identity: bool = False,
                        row_map: torch.Tensor | None = None) -> FeatureSplit:
    """Output buffers of one K4 job (filled by s24_feature_split or by a GEMM's
    background warps via s24_spmm_bg). Its drop statistics are not counted on
    the hot path -- the reference discards them (splitgemm.py:75) -- and are
    recounted on the device only if someone reads them."""
    dev = vals.device
    ns, nd = plan.n_sparse, plan.n_dense
    def recount():
        v, m = (vals, meta_hw) if row_map is None else frame_rows_compressed(vals, meta_hw, row_map, n, h)
        return feature_split(v, m, n, h, plan, with_stats=True).stats._dev

    stats = SparsifyStats(n * ns, recount)
    if identity and not dense_only:
        rows = pad128(2 * nd) + h
        vs = torch.empty(rows, n // 2, dtype=BF16, device=dev)
        es = torch.empty(_lib.meta_hw_bytes(rows, n), dtype=torch.uint8, device=dev)
        return FeatureSplit(vs, es, None, stats, 2 * nd, identity=True)
    paired = paired and not dense_only
    rows = ns + (2 * nd if paired else 0)
    vs = es = vd = None
    if not dense_only:
        vs = torch.empty(max(pad128(rows), 128), n // 2, dtype=BF16, device=dev)
        es = torch.empty(_lib.meta_hw_bytes(max(rows, 1), n), dtype=torch.uint8, device=dev)
    if not paired:
        vd = torch.empty(max(pad128(nd), 128), n, dtype=BF16, device=dev)
    return FeatureSplit(vs, es, vd, stats, 2 * nd if paired else -1)


def run_feature_split(fs: FeatureSplit, vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int,
                      plan: SplitPlan, nonneg: bool = False, row_map: torch.Tensor | None = None) -> None:
    """Fill preallocated K4 outputs on the current stream (no drop counting).
    row_map (paired layout only): token j of the split is row row_map[j] of
    vals / meta_hw (the compute frame's permutation, applied while reading)."""
    if row_map is not None and (fs.identity or fs.pair_rows < 0):
        raise DimensionError("a row-mapped feature split needs the paired rank layout")
    for _ in range(K4_REPEAT):
        if fs.identity:
            _lib.call("s24_feature_split_id", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), plan.n_dense,
                      ptr(fs.vs), ptr(fs.es), None, int(nonneg), stream())
        elif fs.pair_rows >= 0:
            _lib.call("s24_feature_split_x", ptr(vals), None, ptr(meta_hw), n, h, ptr(plan.feat_pos), plan.n_sparse,
                      plan.n_dense, ptr(fs.vs), ptr(fs.es), None, None, int(nonneg), ptr(row_map), stream())
        else:
            _lib.call("s24_feature_split", ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), plan.n_sparse,
                      plan.n_dense, ptr(fs.vs), ptr(fs.es), ptr(fs.vd), None, int(nonneg), fs.pair_rows, stream())


K4_REPEAT = 1  # experiments only (scripts/ab_step.py): marginal cost of K4 in the step


def run_feature_split_dual(fa: FeatureSplit, fb: FeatureSplit, vals_a: torch.Tensor, vals_b: torch.Tensor,
                           meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan,
                           row_map: torch.Tensor | None = None) -> None:
    """K4 for two operands on one keep pattern (the activation, >= 0, and
    g_pre) in one pass: paired rank layout for both."""
    if not (fa.pair_rows >= 0 and fb.pair_rows >= 0 and not fa.identity and not fb.identity):
        raise DimensionError("the dual feature split writes the paired rank layout")
    for _ in range(K4_REPEAT):
        _lib.call("s24_feature_split_x", ptr(vals_a), ptr(vals_b), ptr(meta_hw), n, h, ptr(plan.feat_pos),
                  plan.n_sparse, plan.n_dense, ptr(fa.vs), ptr(fa.es), ptr(fb.vs), ptr(fb.es), 1, ptr(row_map), stream())


def side_stream(device) -> torch.cuda.Stream:
    return _side_stream(device)


def k4_job_args(vals: torch.Tensor, meta_hw: torch.Tensor, n: int, h: int, plan: SplitPlan, fs: FeatureSplit,
                counter: torch.Tensor) -> tuple:
    """The K4 argument tail of s24_spmm_bg (feature split run as background work
    of a sparse GEMM)."""
    return (ptr(vals), ptr(meta_hw), n, h, ptr(plan.feat_pos), plan.n_sparse, plan.n_dense, ptr(fs.vs), ptr(fs.es),
            ptr(fs.vd), ptr(counter))


@dataclass
class FusedFeatureOperand:
    """Feature-wise 2:4 operand of ALL features, written by the K1 / K3
    epilogues: vals bf16 [h, n/2] (K-major along tokens), meta hw (rows = h,
    K = n), counts int64 [h] = nonzeros before | after << 32 per feature."""

    vals: torch.Tensor
    meta: torch.Tensor
    counts: torch.Tensor
    n: int

    @staticmethod
    def alloc(h: int, n: int, device) -> "FusedFeatureOperand":
        return FusedFeatureOperand(torch.empty(pad128(h), n // 2, dtype=BF16, device=device),
                                   torch.empty(_lib.meta_hw_bytes(h, n), dtype=torch.uint8, device=device),
                                   torch.zeros(h, dtype=torch.int64, device=device), n)

    def args(self):
        return ptr(self.vals), ptr(self.meta), ptr(self.counts), self.n

    def stats(self, plan: SplitPlan) -> SparsifyStats:
        """Drop statistics of the sparse partition (what the reference's
        sparsify_feature_wise(am[:, sparse]) would report)."""

        def reduce():
            c = self.counts if plan.n_dense == 0 else self.counts[plan.sparse_features.long()]
            return torch.stack([(c & 0xFFFFFFFF).sum(), (c >> 32).sum()])

        return SparsifyStats(self.n * plan.n_sparse, reduce)


def fused_weight_grad(fo: FusedFeatureOperand, tok_vals: torch.Tensor, tok_meta: torch.Tensor, h: int,
                      plan: SplitPlan, b: torch.Tensor, out: torch.Tensor, transposed: bool) -> None:
    """Split weight gradient from the epilogue-fused feature-wise operand:
    out[S] = sparse GEMM over all h feature rows of `fo` with the dense rows
    skipped in the epilogue (row_valid = feat_pos), out[D] = dense GEMM over
    the dense columns gathered from the token-wise operand (K4 dense-only, on a
    side stream so it overlaps the sparse GEMM)."""
    n = fo.n
    d = b.shape[1]
    ld = out.shape[1]
    code = _lib.F32 if out.dtype == F32 else _lib.BF16
    main = torch.cuda.current_stream()
    if plan.n_dense:
        side = _side_stream(out.device)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            fd = feature_split(tok_vals, tok_meta, n, h, plan, dense_only=True)
            dense_remainder_gemm(fd.vd, b, n, plan, out, transposed, code, side)
    if plan.n_sparse:
        _lib.call("s24_spmm", ptr(fo.vals), ptr(fo.meta), ptr(b), 1, b.stride(0), h, d, n, ptr(out), code, ld, None,
                  int(transposed), h, ptr(plan.feat_pos) if plan.n_dense else None, 0, main.cuda_stream)
    if plan.n_dense:
        main.wait_stream(side)


def split_weight_grad(fs: FeatureSplit, plan: SplitPlan, b: torch.Tensor, n: int, out: torch.Tensor,
                      transposed: bool) -> None:
    """out[S] = sparse(fs)^T b, out[D] = dense(fs)^T b on tensor cores, scattered
    by feature index in the epilogue. b: bf16 [n, d] (K = tokens, MN-major).
    transposed=True writes out as [d, h] (dW1 layout). A paired-layout fs
    (dense features as 2:4 row pairs) needs a single sparse GEMM."""
    d = b.shape[1]
    ld = out.shape[1]
    code = _lib.F32 if out.dtype == F32 else _lib.BF16
    if fs.pair_rows >= 0:
        rows, rmap, valid = fs.gemm_rows(plan)
        if rows:
            _lib.call("s24_spmm", ptr(fs.vs), ptr(fs.es), ptr(b), 1, b.stride(0), rows, d, n, ptr(out), code, ld,
                      ptr(rmap), int(transposed), rows, ptr(valid), fs.pair_rows, stream())
        return
    main = torch.cuda.current_stream()
    side = _side_stream(out.device) if plan.n_sparse and plan.n_dense else main
    if side is not main:
        side.wait_stream(main)  # operands ready; the side work must not wait for the sparse GEMM
    if plan.n_sparse:
        _lib.call("s24_spmm", ptr(fs.vs), ptr(fs.es), ptr(b), 1, b.stride(0), plan.n_sparse, d, n, ptr(out), code,
                  ld, ptr(plan.sparse_features), int(transposed), plan.n_sparse, None, 0, main.cuda_stream)
    if plan.n_dense:
        # the thin dense remainder (~5% of the rows, K = all tokens) is split
        # along K and launched on a side stream right behind the sparse GEMM:
        # its short work units fill the SMs the sparse GEMM's last wave leaves
        # idle; a fixed-order reduction keeps the result deterministic
        with torch.cuda.stream(side):
            dense_remainder_gemm(fs.vd, b, n, plan, out, transposed, code, side)
    if side is not main:
        main.wait_stream(side)


def split_weight_grad_pair(fa: FeatureSplit, fb: FeatureSplit, plan: SplitPlan, b_a: torch.Tensor,
                           b_b: torch.Tensor, n: int, out_a: torch.Tensor, out_b: torch.Tensor) -> None:
    """split_weight_grad for two operands sharing one plan and one (|S|, d, n)
    shape: out_a[S] = sparse(fa)^T b_a (row-major [h, d]) and out_b = (sparse(fb)^T b_b)^T
    (transposed [d, h]) in ONE grouped sparse launch, the two dense
    remainders on the side stream next to it -- or, for paired-layout
    operands, inside the same launch as 2:4 row pairs."""
    d = b_a.shape[1]
    if b_b.shape[1] != d or out_a.dtype != out_b.dtype:
        raise DimensionError("paired weight gradients need equal widths and output dtypes")
    if fa.pair_rows != fb.pair_rows or fa.identity != fb.identity:
        raise DimensionError("both operands must use the same layout")
    code = _lib.F32 if out_a.dtype == F32 else _lib.BF16
    if fa.pair_rows >= 0:
        rows, rmap, valid = fa.gemm_rows(plan)
        rm, rv = ptr(rmap), ptr(valid)
        if rows:
            _lib.call("s24_spmm_pair", 1, rows, d, n, code,
                      ptr(fa.vs), ptr(fa.es), ptr(b_a), b_a.stride(0), ptr(out_a), out_a.shape[1], rm, 0, rv,
                      ptr(fb.vs), ptr(fb.es), ptr(b_b), b_b.stride(0), ptr(out_b), out_b.shape[1], rm, 1, rv,
                      fa.pair_rows, stream())
        return
    main = torch.cuda.current_stream()
    side = _side_stream(out_a.device) if plan.n_sparse and plan.n_dense else main
    if side is not main:
        side.wait_stream(main)
    if plan.n_sparse:
        sf = ptr(plan.sparse_features)
        _lib.call("s24_spmm_pair", 1, plan.n_sparse, d, n, code,
                  ptr(fa.vs), ptr(fa.es), ptr(b_a), b_a.stride(0), ptr(out_a), out_a.shape[1], sf, 0, None,
                  ptr(fb.vs), ptr(fb.es), ptr(b_b), b_b.stride(0), ptr(out_b), out_b.shape[1], sf, 1, None, 0,
                  main.cuda_stream)
    if plan.n_dense:
        with torch.cuda.stream(side):
            dense_remainder_gemm(fa.vd, b_a, n, plan, out_a, False, code, side)
            dense_remainder_gemm(fb.vd, b_b, n, plan, out_b, True, code, side)
    if side is not main:
        main.wait_stream(side)


def dense_remainder_gemm(vd, b, n, plan, out, transposed, code, st) -> None:
    d = b.shape[1]
    nd = plan.n_dense
    k_splits = max(1, min(8, n // 2048))
    if k_splits > 1:
        ws = torch.empty(k_splits, nd, d, dtype=F32, device=out.device)
        _lib.call("s24_gemm_splitk", ptr(vd), 0, n, ptr(b), 1, b.stride(0), nd, d, n, k_splits, ptr(ws), ptr(out),
                  code, out.shape[1], ptr(plan.dense_features), int(transposed), st.cuda_stream)
    else:
        _lib.call("s24_gemm", ptr(vd), 0, n, ptr(b), 1, b.stride(0), nd, d, n, ptr(out), code, out.shape[1],
                  ptr(plan.dense_features), int(transposed), nd, None, st.cuda_stream)


_side_streams: dict[int, torch.cuda.Stream] = {}


def _side_stream(device) -> torch.cuda.Stream:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    st = _side_streams.get(idx)
    if st is None:
        st = _side_streams[idx] = torch.cuda.Stream(device=device)
    return st


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
