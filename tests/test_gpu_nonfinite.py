"""Non-finite values and the masked feature-wise sparsifier on the GPU.

The reference accepts NaN / Inf in the FFN input and weights (ffn_forward and
the sparsifiers check shapes and dtypes only) and handles them with numpy's
semantics: relu keeps NaN (ffn.py:167-169), a NaN counts as a nonzero
(splitgemm.py:28-30) and ranks below every number including zero in the
top-2 (sparse24.py:72-77), Inf ranks above all, and the sparse GEMMs never
multiply entries outside the keep pattern (sparse24.py:170-216). K1, the
token-wise / feature-wise sparsifiers, K4 and the 2:4 tensor-core GEMMs
reproduce that: masks, metadata, counts, plan and drop counts bit for bit,
and outputs with the same non-finite pattern and finite values within the
bf16 tolerance. Fixtures: tests/golden/nonfinite.npz, made by the reference
itself (oracle/make_golden.py)."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def nf():
    return np.load(GOLD / "nonfinite.npz")


def same_nonfinite_close(got, want, tol):
    """identical NaN / +Inf / -Inf positions, finite entries within tol
    (relative Frobenius norm over the finite entries)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    for pred in (np.isnan, np.isposinf, np.isneginf):
        assert np.array_equal(pred(got), pred(want)), pred.__name__
    fin = np.isfinite(want)
    d = got[fin] - want[fin]
    assert np.linalg.norm(d) <= tol * max(np.linalg.norm(want[fin]), 1e-30)


def test_sparsifiers_nonfinite_bitwise(nf):
    for i in range(2):
        a = torch.from_numpy(nf[f"tok{i}_a"]).cuda()
        s, mask, st = s24.sparsify_token_wise(a)
        assert np.array_equal(s.values.float().cpu().numpy(), O.bf16_round(nf[f"tok{i}_values"]), equal_nan=True)
        assert np.array_equal(s.meta.cpu().numpy(), nf[f"tok{i}_meta"])
        assert np.array_equal(mask.cpu().numpy(), nf[f"tok{i}_mask"])
        assert [st.total_entries, st.nonzeros_before, st.nonzeros_after, st.dropped] == nf[f"tok{i}_stats"].tolist()
        f, _, fst = s24.sparsify_feature_wise(a)
        assert np.array_equal(f.values.float().cpu().numpy(), O.bf16_round(nf[f"feat{i}_values"]), equal_nan=True)
        assert np.array_equal(f.meta.cpu().numpy(), nf[f"feat{i}_meta"])
        assert [fst.total_entries, fst.nonzeros_before, fst.nonzeros_after, fst.dropped] == \
            nf[f"feat{i}_stats"].tolist()
        counts = s24.column_nonzero_counts(a)
        assert np.array_equal(counts.cpu().numpy(), nf[f"counts{i}"])
        plan = s24.partition_features(counts, 0.75)
        assert np.array_equal(plan.sparse_features.cpu().numpy(), nf[f"plan{i}_sparse"])


def test_ffn_nonfinite_matches_reference(nf):
    """The reference's own run on NaN / Inf weights and a NaN input row (the
    padded compatibility path: d = 8, h = 16)."""
    cfg = s24.RECIPE
    p = s24.FfnParams(w1=torch.from_numpy(nf["ffn_w1"]).cuda(), w2=torch.from_numpy(nf["ffn_w2"]).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(nf["ffn_x"]).cuda(), p, cfg, keep_pre_act=True)
    g = s24.ffn_backward(torch.from_numpy(nf["ffn_g"]).cuda(), cache, p, cfg)
    torch.cuda.synchronize()
    # the selection on the device's own pre-activation (tensor-core sums may
    # differ from the ordered reference in the last bit, never in NaN / Inf)
    pre = cache.pre_act.cpu().numpy()
    same_nonfinite_close(pre, nf["ffn_pre"], 1e-5)
    r = np.maximum(pre, np.float32(0))
    _, om, omask, ost = O.sparsify_token(r * r)
    assert np.array_equal(cache.fwd_mask.cpu().numpy(), omask)
    assert np.array_equal(cache.fwd_mask.cpu().numpy(), nf["ffn_mask"])
    assert np.array_equal(cache.counts.cpu().numpy(), O.column_counts(r * r))
    st = cache.stats
    assert [st.total_entries, st.nonzeros_before, st.nonzeros_after, st.dropped] == nf["ffn_stats"].tolist()
    assert np.array_equal(cache.plan.sparse_features.cpu().numpy(), nf["ffn_plan_sparse"])
    same_nonfinite_close(out.float().cpu().numpy(), nf["ffn_out"], 1e-2)
    same_nonfinite_close(g.d_x.float().cpu().numpy(), nf["ffn_d_x"], 1e-2)
    same_nonfinite_close(g.d_w1.cpu().numpy(), nf["ffn_d_w1"], 8e-3)
    same_nonfinite_close(g.d_w2.cpu().numpy(), nf["ffn_d_w2"], 8e-3)


def test_ffn_nonfinite_device_tiled_shape():
    """NaN / Inf on a shape the device GEMMs tile directly (no padding):
    K1's NaN semantics, the NaN-aware K4 of the activation (K1 raised its
    flag) and the exact-skip 2:4 GEMMs, against the oracle run on the same
    bf16 inputs."""
    n, d, h = 512, 64, 256
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.8, seed=9)
    w1[:, 3] = np.nan          # a NaN feature: NaN in every token's group
    w1[:, 68:71] = np.nan      # three NaN features in one group: a NaN gets kept
    w1[5, 100] = np.inf
    x[11, 4] = np.nan          # a NaN token
    cfg = s24.RECIPE
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, cfg, keep_pre_act=True)
    g = s24.ffn_backward(torch.from_numpy(dy).cuda(), cache, p, cfg)
    torch.cuda.synchronize()
    assert int(cache.stats_dev[2]) == 1  # NaN among the kept values
    pre = cache.pre_act.cpu().numpy()
    r = np.maximum(pre, np.float32(0))
    act = r * r
    ov, om, omask, ost = O.sparsify_token(act)
    assert np.array_equal(cache.act_sparse.meta.cpu().numpy(), om)
    assert np.array_equal(cache.act_sparse.values.float().cpu().numpy(), O.bf16_round(ov), equal_nan=True)
    assert np.array_equal(cache.counts.cpu().numpy(), O.column_counts(act))
    assert cache.stats.nonzeros_before == ost["nonzeros_before"] and cache.stats.dropped == ost["dropped"]
    osp, ode = O.partition(O.column_counts(act), cfg.split_ratio)
    assert np.array_equal(cache.plan.sparse_features.cpu().numpy(), osp)
    # feature-wise splits on the device's stored values: bit for bit
    act_kept = s24.decompress(cache.act_sparse).cpu().numpy()
    _, _, _, fst = O.sparsify_feature(np.ascontiguousarray(act_kept[:, osp]))
    assert g.stats_act.nonzeros_before == fst["nonzeros_before"] and g.stats_act.dropped == fst["dropped"]
    # end to end against the oracle on the same inputs (mask flips aside, the
    # NaN / Inf pattern is structural)
    ocfg = dict(O.RECIPE)
    with np.errstate(all="ignore"):
        o_out, o_cache = O.ffn_forward(x, w1, w2, ocfg, ordered=False)
        o_g = O.ffn_backward(dy, o_cache, w1, w2, ocfg, ordered=False)
    if np.array_equal(o_cache["mask"], omask):
        same_nonfinite_close(out.float().cpu().numpy(), o_out, 1e-2)
        same_nonfinite_close(g.d_x.float().cpu().numpy(), o_g["d_x"], 1e-2)
        same_nonfinite_close(g.d_w1.cpu().numpy(), o_g["d_w1"], 8e-3)
        same_nonfinite_close(g.d_w2.cpu().numpy(), o_g["d_w2"], 8e-3)


def test_masked_feature_wise_matches_reference(nf):
    """sparsify_feature_wise_masked (ref sparse24.py:118-129) on the device:
    the reference's KATs (tests/test_sparse24.py:119-140) and random masks."""
    for tag in ("ones", "zeros", "r0", "r1", "r2", "r3"):
        a = torch.from_numpy(nf[f"masked_{tag}_a"]).cuda()
        mask = torch.from_numpy(nf[f"masked_{tag}_mask"]).cuda()
        sm, keep, st = s24.sparsify_feature_wise_masked(a, mask)
        assert np.array_equal(sm.values.float().cpu().numpy(), O.bf16_round(nf[f"masked_{tag}_values"]))
        assert np.array_equal(sm.meta.cpu().numpy(), nf[f"masked_{tag}_meta"])
        assert [st.total_entries, st.nonzeros_before, st.nonzeros_after, st.dropped] == \
            nf[f"masked_{tag}_stats"].tolist()
        if tag.startswith("r"):
            assert np.array_equal(keep.cpu().numpy(), nf[f"masked_{tag}_keep"])
        dense = s24.decompress(sm).cpu().numpy()
        assert not np.any(dense[~nf[f"masked_{tag}_mask"]] != 0)  # support inside the mask
    with pytest.raises(s24.DimensionError):
        s24.sparsify_feature_wise_masked(torch.zeros(8, 8, device="cuda"), torch.ones(4, 8, device="cuda"))
    # device-sized: identical to masking first, then the plain feature-wise kernel
    a = torch.randn(512, 384, device="cuda")
    mask = torch.rand(512, 384, device="cuda") < 0.5
    sm, _, st = s24.sparsify_feature_wise_masked(a, mask)
    sp, _, st2 = s24.sparsify_feature_wise(torch.where(mask, a, 0))
    assert torch.equal(sm.data, sp.data) and torch.equal(sm.meta_hw, sp.meta_hw)
    assert (st.nonzeros_before, st.nonzeros_after) == (st2.nonzeros_before, st2.nonzeros_after)
