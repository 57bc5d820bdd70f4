"""Seeded random shapes and values through the drop-in's building blocks
(ref pkg/src/srelu24/__init__.py:7-91) against the oracle: the three
sparsifiers, masked compression and decompression, the 2:4 GEMMs, the split
GEMM with its device plan, and the permutations. Inputs are fp32 or bf16
with exact zeros, ties and (for the sparsifiers) NaN / Inf; shapes include
rows / columns that are not multiples of the device tiles.

Bars: selections, metadata, masks, statistics, counts, plans and
permutations bit-exact; kept values bit-exact after bf16 rounding (the
device stores bf16); GEMMs within 1e-5 relative of the oracle's fp32
reduction over the same (bf16-valued) kept operands.
"""

import os

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu

# S24_FUZZ_SCALE=k runs k times as many seeded cases (ad-hoc campaigns)
SCALE = int(os.environ.get("S24_FUZZ_SCALE", "1"))


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def values(rng, rows, cols, nonfinite=False):
    """bf16-valued fp32: ~40% exact zeros, coarse values (frequent ties)"""
    a = rng.standard_normal((rows, cols)).astype(np.float32)
    a[rng.random((rows, cols)) < 0.4] = 0
    ties = rng.random((rows, cols)) < 0.2
    a[ties] = np.where(rng.random(int(ties.sum())) < 0.5, 1.0, -1.0)
    if nonfinite:
        a[rng.random((rows, cols)) < 0.01] = np.nan
        a[rng.random((rows, cols)) < 0.005] = np.inf
        a[rng.random((rows, cols)) < 0.005] = -np.inf
    return O.bf16_round(a)


def dev(a, bf16):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.bfloat16() if bf16 else t


def shape(rng):
    return int(rng.integers(1, 80)) * 4, int(rng.integers(1, 80)) * 4


@pytest.mark.parametrize("i", range(16 * SCALE))
def test_sparsifiers_and_compression(i):
    rng = np.random.Generator(np.random.PCG64(300 + i))
    rows, cols = shape(rng)
    bf16 = bool(i % 2)
    a = values(rng, rows, cols, nonfinite=i % 4 == 3)
    ta = dev(a, bf16)

    s, mask, st = s24.sparsify_token_wise(ta)
    ov, om, omask, ost = O.sparsify_token(a)
    assert np.array_equal(s.meta.cpu().numpy(), om)
    assert np.array_equal(s.values.float().cpu().numpy(), O.bf16_round(ov), equal_nan=True)
    assert np.array_equal(mask.cpu().numpy(), omask)
    assert (st.nonzeros_before, st.nonzeros_after) == (ost["nonzeros_before"], ost["nonzeros_after"])

    sf, fmask, fst = s24.sparsify_feature_wise(ta)
    fv, fm, fom, fost = O.sparsify_feature(a)
    assert np.array_equal(sf.meta.cpu().numpy(), fm)
    assert np.array_equal(sf.values.float().cpu().numpy(), O.bf16_round(fv), equal_nan=True)
    assert np.array_equal(fmask.cpu().numpy(), fom)
    assert (fst.nonzeros_before, fst.nonzeros_after) == (fost["nonzeros_before"], fost["nonzeros_after"])

    # masked feature-wise on the token-wise mask (ref sparse24.py:118-129)
    smf, mmask, mst = s24.sparsify_feature_wise_masked(ta, mask)
    mv, mm, mom, most = O.sparsify_feature_masked(a, omask)
    assert np.array_equal(smf.meta.cpu().numpy(), mm)
    assert np.array_equal(mmask.cpu().numpy(), mom)
    assert (mst.nonzeros_before, mst.dropped) == (most["nonzeros_before"], most["dropped"])

    # exact compression on the token-wise mask, and back
    c = s24.compress_token_wise_with_mask(ta, mask)
    cv, cm = O.compress_with_mask(a, omask)
    assert np.array_equal(c.meta.cpu().numpy(), cm)
    assert np.array_equal(c.values.float().cpu().numpy(), O.bf16_round(cv), equal_nan=True)
    back = s24.decompress(c).cpu().numpy()
    assert np.array_equal(back, O.bf16_round(np.where(omask, a, np.float32(0))), equal_nan=True)


@pytest.mark.parametrize("i", range(12 * SCALE))
def test_sparse_gemms_split_gemm_and_plan(i):
    rng = np.random.Generator(np.random.PCG64(500 + i))
    rows, cols = shape(rng)
    n_b = int(rng.choice([8, 32, 40, 64, 96]))
    bf16 = bool(i % 2)
    a = values(rng, rows, cols)
    ta = dev(a, bf16)

    # token-wise A [rows, cols] @ B [cols, n_b]
    b = O.bf16_round(rng.standard_normal((cols, n_b)).astype(np.float32))
    s, mask, _ = s24.sparsify_token_wise(ta)
    got = s24.sp_gemm(s, dev(b, True)).cpu().numpy()
    keep = mask.cpu().numpy()
    want = O.gemm_kept(O.bf16_round(np.where(keep, a, np.float32(0))), keep, b, ordered=False)
    assert rel(got, want) < 1e-5

    # feature-wise A: A^T [cols, rows] @ B [rows, n_b]
    bt = O.bf16_round(rng.standard_normal((rows, n_b)).astype(np.float32))
    sf, fmask, _ = s24.sparsify_feature_wise(ta)
    got = s24.sp_gemm_t(sf, dev(bt, True)).cpu().numpy()
    fkeep = fmask.cpu().numpy()
    want = O.gemm_at_kept(O.bf16_round(np.where(fkeep, a, np.float32(0))), fkeep, bt, ordered=False)
    assert rel(got, want) < 1e-5

    # counts, device plan and the split GEMM on the token-wise mask
    ratio = float(rng.choice([0.5, 0.8, 0.95, 1.0]))
    am = np.where(keep, a, np.float32(0))
    counts = s24.column_nonzero_counts(dev(am, bf16))
    assert np.array_equal(counts.cpu().numpy(), O.column_counts(am))
    plan = s24.partition_features(counts, ratio)
    osp, ode = O.partition(O.column_counts(am), ratio)
    assert np.array_equal(plan.sparse_features.cpu().numpy(), osp)
    assert np.array_equal(plan.dense_features.cpu().numpy(), ode)
    got = s24.split_gemm_t(ta, mask, dev(bt, True), plan).cpu().numpy()
    want, _ = O.split_gemm_t(O.bf16_round(a), keep, bt, osp, ode, ordered=False)
    assert rel(got, want) < 1e-5


@pytest.mark.parametrize("i", range(6 * SCALE))
def test_permutations(i):
    rng = np.random.Generator(np.random.PCG64(700 + i))
    n, d = int(rng.integers(1, 300)), int(rng.choice([8, 16, 40, 64]))
    seed = int(rng.integers(0, 10_000))
    p = s24.make_permutation(seed, n)
    op = O.make_permutation(seed, n)
    assert np.array_equal(np.asarray(p.cpu() if torch.is_tensor(p) else p), op)
    a = O.bf16_round(rng.standard_normal((n, d)).astype(np.float32))
    ta = dev(a, True)
    assert np.array_equal(s24.permute_rows(ta, op).float().cpu().numpy(), O.permute_rows(a, op))
    assert np.array_equal(s24.inverse_permute_rows(ta, op).float().cpu().numpy(), O.inverse_permute_rows(a, op))
