"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference 2:4 path.

Every function cites the reference rule it restates
(ref = /root/reference/pkg/src/srelu24/). It is the checker for the CUDA path
and the CPU baseline timed by bench.py; it is never imported by the product
package. Pinned against the reference's own outputs in tests/golden/.

Conventions: plain 2-D numpy arrays in float32 ("working") or float64
("oracle"); compressed matrices are returned as tuples
(values, meta) with the reference's storage layouts:
  token-wise   values/meta [rows, cols/4, 2]   (sparse24.py:30-47)
  feature-wise values/meta [rows/4, cols, 2]
Stats are dicts with the SparsifyStats field names (sparse24.py:50-69).
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------- GEMMs


def gemm(a: np.ndarray, b: np.ndarray, ordered: bool = True) -> np.ndarray:
    """a @ b. ordered=True reproduces the reference's accumulation: one
    rank-1 update per reduction index, ascending, rounded in the operand
    precision after each multiply and add (ref matcore.py:71-87). ordered=False
    uses BLAS (fast, tolerance-level agreement only)."""
    if not ordered:
        return np.matmul(a, b)
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
    for k in range(a.shape[1]):
        acc += np.multiply.outer(a[:, k], b[k])
    return acc


def gemm_at(a: np.ndarray, b: np.ndarray, ordered: bool = True) -> np.ndarray:
    """a.T @ b with reduction over rows of a, ascending (ref matcore.py:90-106)."""
    if not ordered:
        return np.matmul(a.T, b)
    acc = np.zeros((a.shape[1], b.shape[1]), dtype=a.dtype)
    for k in range(a.shape[0]):
        acc += np.multiply.outer(a[k], b[k])
    return acc


def gemm_kept(a: np.ndarray, keep: np.ndarray, b: np.ndarray, ordered: bool = True) -> np.ndarray:
    """sum over kept k of a[:, k] b[k] -- the reference's exact-skip sparse
    product (sp_gemm, ref sparse24.py:170-192: entries outside the keep
    pattern are never multiplied, so a non-finite b row meets only the kept
    entries; kept zeros do multiply). Ascending k when ordered."""
    if not ordered and np.all(np.isfinite(b)):
        return np.matmul(np.where(keep, a, a.dtype.type(0)), b)
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
    with np.errstate(invalid="ignore", over="ignore"):
        for k in range(a.shape[1]):
            rows = keep[:, k]
            if rows.any():
                acc[rows] += np.multiply.outer(a[rows, k], b[k])
    return acc


def gemm_at_kept(a: np.ndarray, keep: np.ndarray, b: np.ndarray, ordered: bool = True) -> np.ndarray:
    """a^T b over kept entries only (sp_gemm_t, ref sparse24.py:195-216)."""
    return gemm_kept(np.ascontiguousarray(a.T), np.ascontiguousarray(keep.T), b, ordered)


# ---------------------------------------------------------------- 2:4 selection

_LOWER = np.arange(4)[:, None] < np.arange(4)[None, :]


def keep_mask4(groups: np.ndarray) -> np.ndarray:
    """Keep mask over the last axis (size 4): the two largest |x|, ties to the
    lower index, zeros last (padding = lowest-index zeros), NaN below all.
    Restates the stable argsort rule of ref sparse24.py:72-77 as a rank test:
    x_i is kept iff fewer than two x_j beat it (|x_j| > |x_i|, or equal with
    j < i)."""
    key = np.where(np.isnan(groups), -1.0, np.abs(groups.astype(np.float64)))
    kj = key[..., :, None]
    ki = key[..., None, :]
    beats = (kj > ki) | ((kj == ki) & _LOWER)
    return beats.sum(axis=-2) < 2


def _positions(keep: np.ndarray) -> np.ndarray:
    """ascending kept positions (i0, i1) of a [..., 4] keep mask."""
    i0 = np.argmax(keep, axis=-1)
    i1 = 3 - np.argmax(keep[..., ::-1], axis=-1)
    return np.stack([i0, i1], axis=-1).astype(np.uint8)


def _stats(total: int, before: int, after: int) -> dict:
    """ref sparse24.py:60-69"""
    dropped = before - after
    return {
        "total_entries": total,
        "nonzeros_before": before,
        "nonzeros_after": after,
        "dropped": dropped,
        "sparsity_before": 1.0 - before / total if total else 0.0,
        "dropped_fraction_of_nonzeros": dropped / before if before else 0.0,
    }


def sparsify_token(a: np.ndarray):
    """Top-2 per group of 4 along rows (ref sparse24.py:80-93).
    Returns (values [r, c/4, 2], meta [r, c/4, 2], mask [r, c], stats)."""
    r, c = a.shape
    if c % 4:
        raise ValueError("cols % 4 != 0")
    g = a.reshape(r, c // 4, 4)
    keep = keep_mask4(g)
    meta = _positions(keep)
    vals = np.take_along_axis(g, meta.astype(np.int64), axis=2)
    return vals, meta, keep.reshape(r, c), _stats(a.size, int(np.count_nonzero(a)), int(np.count_nonzero(vals)))


def sparsify_feature(a: np.ndarray):
    """Top-2 per group of 4 consecutive rows down each column (ref
    sparse24.py:96-115). Returns (values [r/4, c, 2], meta [r/4, c, 2],
    mask [r, c], stats)."""
    r, c = a.shape
    if r % 4:
        raise ValueError("rows % 4 != 0")
    g = np.ascontiguousarray(a.reshape(r // 4, 4, c).transpose(0, 2, 1))  # [r/4, c, 4]
    keep = keep_mask4(g)
    meta = _positions(keep)
    vals = np.take_along_axis(g, meta.astype(np.int64), axis=2)
    mask = keep.transpose(0, 2, 1).reshape(r, c)
    return vals, meta, mask, _stats(a.size, int(np.count_nonzero(a)), int(np.count_nonzero(vals)))


def sparsify_feature_masked(a: np.ndarray, fwd_mask: np.ndarray):
    """Zero entries outside fwd_mask, then sparsify_feature (ref
    sparse24.py:118-129): masked-out values are not counted as dropped."""
    if fwd_mask.shape != a.shape:
        raise ValueError("mask shape does not match matrix")
    return sparsify_feature(np.where(fwd_mask, a, a.dtype.type(0)))


def compress_with_mask(a: np.ndarray, mask: np.ndarray):
    """Exact token-wise compression on a given 2-of-4 mask (ref
    sparse24.py:138-154). Raises ValueError on a group without exactly 2 bits."""
    r, c = a.shape
    mg = mask.reshape(r, c // 4, 4).astype(bool)
    if not np.all(mg.sum(axis=2) == 2):
        raise ValueError("mask must set exactly 2 bits per group of 4")
    meta = _positions(mg)
    vals = np.take_along_axis(a.reshape(r, c // 4, 4), meta.astype(np.int64), axis=2)
    return vals, meta


def decompress_token(vals: np.ndarray, meta: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """ref sparse24.py:157-161"""
    out = np.zeros((rows, cols // 4, 4), dtype=vals.dtype)
    np.put_along_axis(out, meta.astype(np.int64), vals, axis=2)
    return out.reshape(rows, cols)


def decompress_feature(vals: np.ndarray, meta: np.ndarray, rows: int, cols: int) -> np.ndarray:
    """ref sparse24.py:162-167"""
    out = np.zeros((rows // 4, cols, 4), dtype=vals.dtype)
    np.put_along_axis(out, meta.astype(np.int64), vals, axis=2)
    return np.ascontiguousarray(out.transpose(0, 2, 1)).reshape(rows, cols)


# ---------------------------------------------------------------- e4m3 (fp8)

E4M3_MAX = 448.0


def e4m3_values() -> np.ndarray:
    """float64 value of every code (ref matcore.py:113-145): sign | 4-bit
    exponent (bias 7) | 3-bit mantissa, subnormals at exponent 0, NaN only at
    S.1111.111, no infinities; 0x80 is -0."""
    c = np.arange(256)
    e, m = (c >> 3) & 0xF, c & 7
    mag = np.where(e == 0, m * 2.0**-9, np.ldexp(1.0 + m / 8.0, e - 7))
    v = np.where(c & 0x80, -mag, mag)
    v[(e == 15) & (m == 7)] = np.nan
    return v


_E4M3 = e4m3_values()
_E4M3_F32 = _E4M3.astype(np.float32)
_E4M3_GRID = _E4M3[:127]  # codes 0x00..0x7E: the non-negative finite values, increasing


def e4m3_encode(x) -> np.ndarray:
    """Nearest code, ties to the even code (= even mantissa), magnitudes above
    448 saturate to 0x7E, sign from the sign bit (ref matcore.py:155-197). A
    nearest-neighbour search on the value grid rather than the reference's
    frexp arithmetic; pinned against it in tests/golden/fp8.npz."""
    xf = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(xf)):
        raise ValueError("e4m3_encode requires finite input")
    ax = np.minimum(np.abs(xf), E4M3_MAX)
    hi = np.clip(np.searchsorted(_E4M3_GRID, ax, side="left"), 1, 126)
    lo = hi - 1
    dlo, dhi = ax - _E4M3_GRID[lo], _E4M3_GRID[hi] - ax
    code = np.where(dlo < dhi, lo, np.where(dhi < dlo, hi, np.where(lo % 2 == 0, lo, hi)))
    code = np.where(ax == 0, 0, code)
    return (code | np.where(np.signbit(xf), 0x80, 0)).astype(np.uint8)


def e4m3_scales(amax: np.ndarray) -> np.ndarray:
    """amax / 448 in float32, 1 for zero or underflowing slices (ref
    matcore.py:214-220)."""
    amax = np.asarray(amax, dtype=np.float32)
    s = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    return np.where(s > 0, s, np.float32(1.0)).astype(np.float32)


def quantize(a: np.ndarray, axis: str):
    """Per-row ("rows") or per-column ("cols") e4m3 codes and float32 scales of
    a float32 matrix (ref matcore.py:203-225)."""
    red = 1 if axis == "rows" else 0
    amax = np.max(np.abs(a), axis=red) if a.shape[red] else np.zeros(a.shape[1 - red], np.float32)
    sc = e4m3_scales(amax)
    den = sc[:, None] if axis == "rows" else sc[None, :]
    return e4m3_encode(a / den).reshape(a.shape), sc


def quantize_groups(vals: np.ndarray, axes) -> tuple:
    """Scales over the kept values of a compressed matrix (token-wise: axes
    (1, 2) per row; feature-wise: (0, 2) per column) and the values snapped to
    the e4m3 grid, unscaled (ref ffn.py:221-237)."""
    if vals.size == 0:
        return vals, np.ones(vals.shape[0] if axes == (1, 2) else vals.shape[1], np.float32)
    amax = np.max(np.abs(vals), axis=axes)
    sc = e4m3_scales(amax)
    den = sc[:, None, None] if axes == (1, 2) else sc[None, :, None]
    return _E4M3_F32[e4m3_encode(vals / den)], sc


def mm_f8(a, b, ordered=True):
    """(sa x sb) * (decode(qa) @ decode(qb)), a per row, b per column
    (ref ffn.py:206-209, matcore.py:238-258)."""
    qa, sa = quantize(a, "rows")
    qb, sb = quantize(b, "cols")
    return (sa[:, None] * sb[None, :]) * gemm(_E4M3_F32[qa], _E4M3_F32[qb], ordered)


def mm_at_f8(a, b, ordered=True):
    """a^T b with both operands per column (ref ffn.py:212-218)."""
    qa, sa = quantize(a, "cols")
    qb, sb = quantize(b, "cols")
    return (sa[:, None] * sb[None, :]) * gemm_at(_E4M3_F32[qa], _E4M3_F32[qb], ordered)


def sp_mm_f8(vals, meta, rows, cols, b, ordered=True):
    """token-wise 2:4 (per-row scales) times b (per-column), ref ffn.py:240-246"""
    grid, sr = quantize_groups(vals, (1, 2))
    qb, sb = quantize(b, "cols")
    acc = gemm(decompress_token(grid, meta, rows, cols), _E4M3_F32[qb], ordered)
    return (sr[:, None] * sb[None, :]) * acc


def sp_mm_t_f8(vals, meta, rows, cols, b, ordered=True):
    """feature-wise 2:4 transposed (per-feature scales) times b, ref ffn.py:249-255"""
    grid, sc = quantize_groups(vals, (0, 2))
    qb, sb = quantize(b, "cols")
    acc = gemm_at(decompress_feature(grid, meta, rows, cols), _E4M3_F32[qb], ordered)
    return (sc[:, None] * sb[None, :]) * acc


def split_mm_t_f8(a, mask, b, sparse, dense, ordered=True):
    """ref ffn.py:258-270: masked a; sparse features through sp_mm_t_f8, dense
    features through mm_at_f8 (each quantized on its own slice)."""
    am = np.where(mask, a, a.dtype.type(0))
    out = np.zeros((a.shape[1], b.shape[1]), dtype=a.dtype)
    if len(sparse):
        sub = np.ascontiguousarray(am[:, sparse])
        v, m, _, _ = sparsify_feature(sub)
        out[sparse] = sp_mm_t_f8(v, m, *sub.shape, b, ordered)
    if len(dense):
        out[dense] = mm_at_f8(np.ascontiguousarray(am[:, dense]), b, ordered)
    return out


# ---------------------------------------------------------------- split plan


def column_counts(a: np.ndarray) -> np.ndarray:
    """ref splitgemm.py:28-30"""
    return (a != 0).sum(axis=0).astype(np.int64)


def ceil_fraction(ratio: float, h: int) -> int:
    """ref splitgemm.py:33-38 (integral products guarded against float noise)"""
    x = ratio * h
    return int(round(x)) if abs(x - round(x)) < 1e-9 else math.ceil(x)


def partition(counts: np.ndarray, ratio: float):
    """(sparse, dense) ascending index lists; the ceil(ratio*h) features with
    the smallest (count, index) keys are sparse (ref splitgemm.py:41-52)."""
    counts = np.asarray(counts, dtype=np.int64)
    h = counts.shape[0]
    order = np.lexsort((np.arange(h), counts))
    k = ceil_fraction(ratio, h)
    return np.sort(order[:k]), np.sort(order[k:])


def split_gemm_t(a, mask, b, sparse, dense, ordered=True):
    """Masked a^T b with the sparse features feature-wise 2:4 sparsified
    (ref splitgemm.py:55-81), computed as one ordered a^T b over the composite
    operand (bitwise equal to the reference's two-part evaluation because every
    output row is an independent ascending reduction). Returns (out, stats of
    the feature-wise sparsification)."""
    am = np.where(mask, a, a.dtype.type(0))
    comp = am.copy()
    # dense features: every token multiplies (gemm_at over the masked column,
    # ref splitgemm.py:78-80); sparse features: the feature-wise kept entries
    # only (sp_gemm_t)
    keep = np.ones(am.shape, dtype=bool)
    st = _stats(0, 0, 0)
    if len(sparse):
        sub = np.ascontiguousarray(am[:, sparse])
        v, m, fmask, st = sparsify_feature(sub)
        comp[:, sparse] = decompress_feature(v, m, *sub.shape)
        keep[:, sparse] = fmask
    return gemm_at_kept(comp, keep, b, ordered), st


# ---------------------------------------------------------------- permutation


def make_permutation(seed: int, n: int) -> np.ndarray:
    """Fisher-Yates over a PCG64 stream, swapping from the top (ref
    matcore.py:269-280). The draw sequence rng.integers(0, i + 1) for
    i = n-1 .. 1 is the definition of the permutation."""
    gen = np.random.Generator(np.random.PCG64(seed))
    perm = np.arange(n, dtype=np.int64)
    for i in range(n - 1, 0, -1):
        j = int(gen.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def permute_rows(a, p):
    """out[p[i]] = a[i] (ref matcore.py:291-296)"""
    out = np.empty_like(a)
    out[p] = a
    return out


def inverse_permute_rows(a, p):
    """out[i] = a[p[i]] (ref matcore.py:299-302)"""
    return a[p]


# ---------------------------------------------------------------- FFN

RECIPE = dict(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
              permute_tokens=True, permute_seed=0, split_ratio=0.95)
DENSE = dict(forward_mode="dense", backward_mode="dense", mask_grad_with_fwd=False,
             permute_tokens=False, permute_seed=0, split_ratio=0.95)


def ffn_forward(x, w1, w2, cfg, plan=None, ordered=True):
    """Squared-ReLU FFN forward (ref ffn.py:276-363, squared_relu), with the
    e4m3 emulation when cfg["fp8_emulation"]. Returns (out, cache dict)."""
    n = x.shape[0]
    fp8 = cfg.get("fp8_emulation", False)
    sparse_fwd = cfg["forward_mode"] == "sparse24"
    perm = None
    x_in = x
    if cfg["permute_tokens"] and sparse_fwd:
        perm = make_permutation(cfg["permute_seed"], n)
        x_in = permute_rows(x, perm)
    pre = mm_f8(x_in, w1, ordered) if fp8 else gemm(x_in, w1, ordered)
    r = np.maximum(pre, pre.dtype.type(0))
    act = r * r
    counts = column_counts(act)
    if cfg["backward_mode"] == "split_masked" and plan is None:
        plan = partition(counts, cfg["split_ratio"])
    cache = dict(x_in=x_in, pre=pre, perm=perm, plan=plan, counts=counts, mask=None, vals=None, meta=None,
                 act=None, stats=None)
    if sparse_fwd:
        vals, meta, mask, st = sparsify_token(act)
        if fp8:
            # quantize after selection (ref ffn.py:330-341): the backward sees
            # the dequantized values
            grid, sr = quantize_groups(vals, (1, 2))
            qw2, s2 = quantize(w2, "cols")
            out_c = (sr[:, None] * s2[None, :]) * gemm(decompress_token(grid, meta, *act.shape), _E4M3_F32[qw2],
                                                       ordered)
            vals = grid * sr[:, None, None]
            kept = decompress_token(vals, meta, *act.shape)
        else:
            kept = decompress_token(vals, meta, *act.shape)
            out_c = gemm_kept(kept, mask, w2, ordered)
        cache.update(mask=mask, vals=vals, meta=meta, act=kept, stats=st)
    else:
        out_c = mm_f8(act, w2, ordered) if fp8 else gemm(act, w2, ordered)
        cache.update(act=act)
    out = inverse_permute_rows(out_c, perm) if perm is not None else out_c
    return out, cache


def ffn_backward(g_out, cache, w1, w2, cfg, ordered=True):
    """Six-GEMM backward (ref ffn.py:366-451, squared_relu), e4m3 GEMMs when
    cfg["fp8_backward"]. Returns dict(d_w1, d_w2, d_x, fstats_act, fstats_g)."""
    if cfg.get("fp8_backward", False):
        return _ffn_backward_f8(g_out, cache, w1, w2, cfg, ordered)
    perm = cache["perm"]
    g_c = permute_rows(g_out, perm) if perm is not None else g_out
    g_act = gemm(g_c, np.ascontiguousarray(w2.T), ordered)
    g_pre = g_act * (2 * np.maximum(cache["pre"], cache["pre"].dtype.type(0)))
    if cfg["mask_grad_with_fwd"]:
        g_pre = np.where(cache["mask"], g_pre, g_pre.dtype.type(0))
    act = cache["act"]
    fst_a = fst_g = None
    mode = cfg["backward_mode"]
    if mode == "dense":
        d_w2 = gemm_at(act, g_c, ordered)
        d_w1 = gemm_at(cache["x_in"], g_pre, ordered)
    elif mode == "naive_sparse":
        v, m, km, fst_a = sparsify_feature(act)
        d_w2 = gemm_at_kept(decompress_feature(v, m, *act.shape), km, g_c, ordered)
        v, m, km, fst_g = sparsify_feature(g_pre)
        d_w1 = gemm_at_kept(decompress_feature(v, m, *g_pre.shape), km, cache["x_in"], ordered).T
    else:
        sp, de = cache["plan"]
        d_w2, fst_a = split_gemm_t(act, cache["mask"], g_c, sp, de, ordered)
        d_w1t, fst_g = split_gemm_t(g_pre, cache["mask"], cache["x_in"], sp, de, ordered)
        d_w1 = d_w1t.T
    if cfg["mask_grad_with_fwd"]:
        # compress_token_wise_with_mask + sp_gemm: the mask's entries only (ref ffn.py:440-445)
        d_x_c = gemm_kept(g_pre, cache["mask"], np.ascontiguousarray(w1.T), ordered)
    else:
        d_x_c = gemm(g_pre, np.ascontiguousarray(w1.T), ordered)
    d_x = inverse_permute_rows(d_x_c, perm) if perm is not None else d_x_c
    return dict(d_w1=np.ascontiguousarray(d_w1), d_w2=d_w2, d_x=d_x, g_pre=g_pre, fstats_act=fst_a,
                fstats_g=fst_g)


def _ffn_backward_f8(g_out, cache, w1, w2, cfg, ordered=True):
    """ref ffn.py:389-447 with fp8b: every GEMM through the e4m3 emulation."""
    perm = cache["perm"]
    g_c = permute_rows(g_out, perm) if perm is not None else g_out
    g_act = mm_f8(g_c, np.ascontiguousarray(w2.T), ordered)
    g_pre = g_act * (2 * np.maximum(cache["pre"], cache["pre"].dtype.type(0)))
    if cfg["mask_grad_with_fwd"]:
        g_pre = np.where(cache["mask"], g_pre, g_pre.dtype.type(0))
    act = cache["act"]
    mode = cfg["backward_mode"]
    if mode == "dense":
        d_w2 = mm_at_f8(act, g_c, ordered)
        d_w1 = mm_at_f8(cache["x_in"], g_pre, ordered)
    elif mode == "naive_sparse":
        v, m, _, _ = sparsify_feature(act)
        d_w2 = sp_mm_t_f8(v, m, *act.shape, g_c, ordered)
        v, m, _, _ = sparsify_feature(g_pre)
        d_w1 = sp_mm_t_f8(v, m, *g_pre.shape, cache["x_in"], ordered).T
    else:
        sp, de = cache["plan"]
        d_w2 = split_mm_t_f8(act, cache["mask"], g_c, sp, de, ordered)
        d_w1 = split_mm_t_f8(g_pre, cache["mask"], cache["x_in"], sp, de, ordered).T
    if cfg["mask_grad_with_fwd"]:
        v, m = compress_with_mask(g_pre, cache["mask"])
        d_x_c = sp_mm_f8(v, m, *g_pre.shape, np.ascontiguousarray(w1.T), ordered)
    else:
        d_x_c = mm_f8(g_pre, np.ascontiguousarray(w1.T), ordered)
    d_x = inverse_permute_rows(d_x_c, perm) if perm is not None else d_x_c
    return dict(d_w1=np.ascontiguousarray(d_w1), d_w2=d_w2, d_x=d_x, g_pre=g_pre, fstats_act=None, fstats_g=None)


# ---------------------------------------------------------------- synthetic inputs


def synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=0, dense_frac=0.05, dense_sparsity=0.5):
    """x ~ N(0,1) with a bias-carrier last column of ones; W1 ~ N(0, 1/(d-1))
    with last row = per-feature offsets Phi^-1(1 - s_j) so feature j fires with
    probability ~ 1 - s_j; 95% of features at `sparsity`, 5% at 0.5;
    W2 ~ N(0, 1/h); dY ~ N(0, 1). All rounded to bf16 (returned as float32)."""
    from statistics import NormalDist

    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((n, d)).astype(np.float32)
    x[:, -1] = 1.0
    w1 = (rng.standard_normal((d, h)) / math.sqrt(max(d - 1, 1))).astype(np.float32)
    s = np.full(h, sparsity)
    nd = int(round(dense_frac * h))
    if nd:
        s[rng.choice(h, nd, replace=False)] = dense_sparsity
    nd_ = NormalDist()
    w1[-1, :] = np.array([nd_.inv_cdf(1.0 - si) for si in s], dtype=np.float32)
    w2 = (rng.standard_normal((h, d)) / math.sqrt(h)).astype(np.float32)
    dy = rng.standard_normal((n, d)).astype(np.float32)
    return tuple(bf16_round(t) for t in (x, w1, w2, dy))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """round-to-nearest-even to bfloat16, returned as float32"""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    rounded = ((u.astype(np.uint64) + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint32) << 16
    out = rounded.view(np.float32).copy()
    out[np.isnan(a)] = np.nan
    return out
