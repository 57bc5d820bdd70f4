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
