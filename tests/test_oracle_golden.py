"""Pin the numpy oracle to the reference: every golden vector in tests/golden/
(produced by the reference implementation itself, oracle/make_golden.py)
must be reproduced bit for bit by oracle/srelu24_np.py. CPU only."""

from pathlib import Path

import numpy as np
import pytest

from oracle import srelu24_np as O

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def sp():
    return np.load(GOLD / "sparse24.npz")


@pytest.fixture(scope="module")
def sg():
    return np.load(GOLD / "splitgemm.npz")


@pytest.fixture(scope="module")
def ffn():
    return np.load(GOLD / "ffn.npz")


def _stats(st):
    return [st["total_entries"], st["nonzeros_before"], st["nonzeros_after"], st["dropped"]]


def test_token_wise_kats(sp):
    for i in range(4):
        v, m, mask, st = O.sparsify_token(sp[f"kat{i}_a"])
        assert np.array_equal(v, sp[f"kat{i}_values"])
        assert np.array_equal(m, sp[f"kat{i}_meta"])
        assert np.array_equal(mask, sp[f"kat{i}_mask"])
        assert _stats(st) == sp[f"kat{i}_stats"].tolist()


def test_random_sparsifiers_and_kernels(sp):
    for i in range(3):
        a = sp[f"tok{i}_a"]
        v, m, mask, st = O.sparsify_token(a)
        assert np.array_equal(v, sp[f"tok{i}_values"]) and np.array_equal(m, sp[f"tok{i}_meta"])
        assert np.array_equal(mask, sp[f"tok{i}_mask"]) and _stats(st) == sp[f"tok{i}_stats"].tolist()
        fv, fm, fmask, fst = O.sparsify_feature(a)
        assert np.array_equal(fv, sp[f"feat{i}_values"]) and np.array_equal(fm, sp[f"feat{i}_meta"])
        assert np.array_equal(fmask, sp[f"feat{i}_mask"]) and _stats(fst) == sp[f"feat{i}_stats"].tolist()
        kept = O.decompress_token(v, m, *a.shape)
        cv, cm = O.compress_with_mask(kept, mask)
        assert np.array_equal(cv, sp[f"cmp{i}_values"]) and np.array_equal(cm, sp[f"cmp{i}_meta"])
        # exact-skip sparse GEMMs == ordered dense GEMM on the decompressed operand, bitwise
        assert np.array_equal(O.gemm(kept, sp[f"spg{i}_b"]), sp[f"spg{i}_out"])
        fk = O.decompress_feature(fv, fm, *a.shape)
        assert np.array_equal(O.gemm_at(fk, sp[f"spgt{i}_b"]), sp[f"spgt{i}_out"])


def test_plans(sg):
    i = 0
    while f"plan{i}_counts" in sg:
        sparse, dense = O.partition(sg[f"plan{i}_counts"], float(sg[f"plan{i}_ratio"][0]))
        assert np.array_equal(sparse, sg[f"plan{i}_sparse"]), i
        assert np.array_equal(dense, sg[f"plan{i}_dense"]), i
        i += 1
    assert i >= 10


def test_permutations(sg):
    i = 0
    while f"perm{i}_p" in sg:
        p = sg[f"perm{i}_p"]
        assert np.array_equal(O.make_permutation(int(sg[f"perm{i}_seed"][0]), len(p)), p)
        i += 1


def test_split_gemm_bitwise(sg):
    for i in range(4):
        out, _ = O.split_gemm_t(sg[f"split{i}_a"], sg[f"split{i}_mask"], sg[f"split{i}_b"], sg[f"split{i}_sparse"],
                                sg[f"split{i}_dense"])
        assert np.array_equal(out, sg[f"split{i}_out"])


CONFIGS = {
    "recipe": O.RECIPE,
    "dense": O.DENSE,
    "fwd_sparse": dict(O.DENSE, forward_mode="sparse24"),
    "naive_masked": dict(O.DENSE, forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True),
    "split_nomask": dict(O.DENSE, forward_mode="sparse24", backward_mode="split_masked"),
    "recipe_seed3_r05": dict(O.RECIPE, permute_seed=3, split_ratio=0.5),
}


@pytest.mark.parametrize("shape", ["s0", "s1"])
@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_ffn_forward_backward_bitwise(ffn, shape, name):
    x, w1, w2, g = (ffn[f"{shape}_{k}"] for k in ("x", "w1", "w2", "g"))
    cfg = CONFIGS[name]
    out, cache = O.ffn_forward(x, w1, w2, cfg)
    grads = O.ffn_backward(g, cache, w1, w2, cfg)
    k = f"{shape}_{name}"
    assert np.array_equal(out, ffn[f"{k}_out"])
    for t in ("d_w1", "d_w2", "d_x"):
        assert np.array_equal(grads[t], ffn[f"{k}_{t}"]), t
    if f"{k}_mask" in ffn:
        assert np.array_equal(cache["mask"], ffn[f"{k}_mask"])
        assert _stats(cache["stats"]) == ffn[f"{k}_stats"].tolist()
    if f"{k}_plan_sparse" in ffn:
        assert np.array_equal(cache["plan"][0], ffn[f"{k}_plan_sparse"])


def test_analytic_drop_fraction():
    # iid Bernoulli(p) support: E[dropped]/E[nonzero] = (4p^3(1-p) + 2p^4)/(4p)
    # (ref tests/test_acceptance.py:93-104); ~0.95% at p = 0.1
    p = 0.1
    analytic = (4 * p**3 * (1 - p) + 2 * p**4) / (4 * p)
    a = ((np.random.default_rng(42).random((512, 2048)) < p) * 1.0).astype(np.float32)
    _, _, _, st = O.sparsify_token(a)
    assert abs(st["dropped_fraction_of_nonzeros"] - analytic) < 0.0015


# ---------------------------------------------------------------- e4m3 (fp8)


@pytest.fixture(scope="module")
def f8():
    return np.load(GOLD / "fp8.npz")


def test_e4m3_decode_and_encode_bitwise(f8):
    dec = f8["dec_table"]
    assert np.array_equal(np.isnan(dec), np.isnan(O._E4M3))
    ok = ~np.isnan(dec)
    assert np.array_equal(dec[ok], O._E4M3[ok]) and np.array_equal(np.signbit(dec[ok]), np.signbit(O._E4M3[ok]))
    assert np.array_equal(O.e4m3_encode(f8["enc_x"]), f8["enc_codes"])
    # all 254 non-NaN codes round-trip (ref tests/test_acceptance.py:272-280)
    codes = np.arange(256)[ok]
    assert np.array_equal(O.e4m3_encode(O._E4M3[codes]), codes.astype(np.uint8))


@pytest.mark.parametrize("i", range(3))
@pytest.mark.parametrize("axis", ["rows", "cols"])
def test_quantize_bitwise(f8, i, axis):
    codes, scales = O.quantize(f8[f"q{i}_a"], axis)
    assert np.array_equal(codes, f8[f"q{i}_{axis}_codes"])
    assert np.array_equal(scales, f8[f"q{i}_{axis}_scales"])


def test_fp8_gemm_bitwise_and_error_bound(f8):
    a, b = f8["gemm_a"], f8["gemm_b"]
    out = O.mm_f8(a, b)
    assert np.array_equal(out, f8["gemm_out"])
    ref = a.astype(np.float64) @ b.astype(np.float64)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 0.06  # ref tests/test_acceptance.py:283-291


F8_CONFIGS = {
    "recipe_f8fwd": dict(O.RECIPE, fp8_emulation=True),
    "recipe_f8all": dict(O.RECIPE, fp8_emulation=True, fp8_backward=True),
    "dense_f8all": dict(O.DENSE, fp8_emulation=True, fp8_backward=True),
    "naive_f8all": dict(O.DENSE, forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True,
                        fp8_emulation=True, fp8_backward=True),
    "split_nomask_f8all": dict(O.DENSE, forward_mode="sparse24", backward_mode="split_masked", fp8_emulation=True,
                               fp8_backward=True),
}


@pytest.mark.parametrize("shape", ["s0", "s1"])
@pytest.mark.parametrize("name", sorted(F8_CONFIGS))
def test_fp8_ffn_bitwise(f8, shape, name):
    x, w1, w2, g = (f8[f"{shape}_{k}"] for k in ("x", "w1", "w2", "g"))
    cfg = F8_CONFIGS[name]
    out, cache = O.ffn_forward(x, w1, w2, cfg)
    grads = O.ffn_backward(g, cache, w1, w2, cfg)
    k = f"{shape}_{name}"
    assert np.array_equal(out, f8[f"{k}_out"])
    for t in ("d_w1", "d_w2", "d_x"):
        assert np.array_equal(grads[t], f8[f"{k}_{t}"]), t
    if f"{k}_act_values" in f8:
        assert np.array_equal(cache["vals"], f8[f"{k}_act_values"])


def test_fp8_selects_before_quantizing(f8):
    # ref tests/test_ffn.py:360-367: 3.01, 3.0, 2.99 share one code, the
    # selection still keeps the two largest unquantized values
    eye = np.eye(4, dtype=np.float32)
    _, cache = O.ffn_forward(f8["kat_sel_x"], eye, eye, dict(O.DENSE, forward_mode="sparse24", fp8_emulation=True))
    assert np.array_equal(cache["meta"], f8["kat_sel_meta"])


@pytest.fixture(scope="module")
def nf():
    return np.load(GOLD / "nonfinite.npz")


def test_nonfinite_selection_counts_and_plan(nf):
    """NaN / Inf as the reference treats them (fixtures from the reference
    itself): NaN ranks below zero, counts as a nonzero, Inf ranks above all."""
    for i in range(2):
        a = nf[f"tok{i}_a"]
        v, m, mask, st = O.sparsify_token(a)
        assert np.array_equal(v, nf[f"tok{i}_values"], equal_nan=True)
        assert np.array_equal(m, nf[f"tok{i}_meta"]) and np.array_equal(mask, nf[f"tok{i}_mask"])
        assert _stats(st) == nf[f"tok{i}_stats"].tolist()
        fv, fm, _, fst = O.sparsify_feature(a)
        assert np.array_equal(fv, nf[f"feat{i}_values"], equal_nan=True)
        assert np.array_equal(fm, nf[f"feat{i}_meta"]) and _stats(fst) == nf[f"feat{i}_stats"].tolist()
        counts = O.column_counts(a)
        assert np.array_equal(counts, nf[f"counts{i}"])
        assert np.array_equal(O.partition(counts, 0.75)[0], nf[f"plan{i}_sparse"])


def test_nonfinite_ffn(nf):
    cfg = dict(O.RECIPE)
    with np.errstate(all="ignore"):
        out, cache = O.ffn_forward(nf["ffn_x"], nf["ffn_w1"], nf["ffn_w2"], cfg)
        g = O.ffn_backward(nf["ffn_g"], cache, nf["ffn_w1"], nf["ffn_w2"], cfg)
    assert np.array_equal(cache["mask"], nf["ffn_mask"])
    assert np.array_equal(cache["plan"][0], nf["ffn_plan_sparse"])
    assert np.array_equal(out, nf["ffn_out"], equal_nan=True)
    for k in ("d_x", "d_w1", "d_w2"):
        assert np.array_equal(g[k], nf[f"ffn_{k}"], equal_nan=True), k


def test_masked_feature_wise_kats(nf):
    """ref tests/test_sparse24.py:119-140: all-ones mask = plain feature-wise,
    all-zeros mask removes everything and drops nothing, support stays inside
    the mask; plus random masks against the reference's own outputs."""
    for tag in ("ones", "zeros"):
        v, m, _, st = O.sparsify_feature_masked(nf[f"masked_{tag}_a"], nf[f"masked_{tag}_mask"])
        assert np.array_equal(v, nf[f"masked_{tag}_values"]) and np.array_equal(m, nf[f"masked_{tag}_meta"])
        assert _stats(st) == nf[f"masked_{tag}_stats"].tolist()
    assert nf["masked_zeros_stats"].tolist()[1:] == [0, 0, 0]
    for i in range(4):
        a, mask = nf[f"masked_r{i}_a"], nf[f"masked_r{i}_mask"]
        v, m, keep, st = O.sparsify_feature_masked(a, mask)
        assert np.array_equal(v, nf[f"masked_r{i}_values"]) and np.array_equal(m, nf[f"masked_r{i}_meta"])
        assert np.array_equal(keep, nf[f"masked_r{i}_keep"]) and _stats(st) == nf[f"masked_r{i}_stats"].tolist()
        assert not np.any(O.decompress_feature(v, m, *a.shape)[~mask] != 0)
