"""Parity at BASELINE's full sizes -- c2 (n = 16384, d = 2048, h = 8192) and
the 7B-class c4 shape (n = 32768, d = 4096, h = 16384) at activation sparsity
0.9 and at the c5 sweep's extremes 0.5 and 0.98: the recipe fwd + bwd on the
device vs the reference's rules restated in PyTorch (ref ffn.py:276-451,
sparse24.py:72-115, splitgemm.py:28-81) on the same GPU. The numpy oracle is
too slow at these sizes; the torch restatement follows it rule for rule and
is itself checked against the oracle at small size below.

Checks (size-independent properties plus stated tolerances):
* token-wise keep mask: exactly 2 per group of 4, and a top-2 of the fp32
  relu^2 (bitwise against the rank rule on the device's own pre-activation);
* kept values = bf16(act) at the kept positions, bitwise;
* per-feature counts, drop statistics and the split plan: bitwise;
* K4's feature-wise operands of act AND g_pre, every feature (the dense ones
  as row pairs): values and metadata bitwise against the rank rule applied
  to the device's own stored bf16 act / g_pre; both splits' drop counts
  (stats_act, stats_grad) bitwise;
* out, dX (bf16) rel. Frobenius <= 1e-2; dW1, dW2 (fp32) <= 8e-3 against the
  fp32 restatement, mask flips from accumulation order <= 1e-4 of entries.
"""

import math

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(float(b.norm()), 1e-30))


def top2_mask(a4: torch.Tensor) -> torch.Tensor:
    """Rank rule over the last axis (size 4): keep x_i iff fewer than two x_j
    beat it (|x_j| > |x_i|, or equal with j < i); NaN below everything."""
    key = torch.where(torch.isnan(a4), torch.full_like(a4, -1.0), a4.abs())
    kj, ki = key.unsqueeze(-1), key.unsqueeze(-2)  # [..., j, i]
    lower = torch.arange(4, device=a4.device)[:, None] < torch.arange(4, device=a4.device)[None, :]
    beats = (kj > ki) | ((kj == ki) & lower)
    return beats.sum(dim=-2) < 2


def feature_top2(a: torch.Tensor) -> torch.Tensor:
    """Feature-wise 2:4 (groups of 4 consecutive rows down each column), dense."""
    n, c = a.shape
    g = a.reshape(n // 4, 4, c).transpose(1, 2)  # [n/4, c, 4]
    return (g * top2_mask(g)).transpose(1, 2).reshape(n, c)


def plan_lists(counts: torch.Tensor, ratio: float):
    h = counts.numel()
    k = O.ceil_fraction(ratio, h)
    order = np.lexsort((np.arange(h), counts.cpu().numpy()))
    return np.sort(order[:k]), np.sort(order[k:])


def torch_recipe(x, w1, w2, dy, perm, mask_dev=None, act_store=None, g_store=None):
    """fp32 torch restatement of the recipe forward + backward (TF32 off).
    act_store / g_store (optional [n, h] images of the device's stored bf16
    act and g_pre): the feature-wise splits of the weight gradients select on
    and multiply those values -- the selection itself is checked bitwise
    elsewhere, so the comparison isolates the GEMMs' arithmetic from selection
    flips caused by the bf16 storage of act / g_pre."""
    inv = torch.from_numpy(np.argsort(perm)).to(x.device)  # out[i] = a[perm[i]] <=> x_in = x[inv]
    x_in = x.float()[inv]
    pre = x_in @ w1.float()
    act = torch.clamp_min(pre, 0) ** 2
    n, h = act.shape
    mask = top2_mask(act.reshape(n, h // 4, 4)).reshape(n, h) if mask_dev is None else mask_dev
    kept = act * mask
    out_c = kept @ w2.float()
    out = out_c[torch.from_numpy(perm).to(x.device)]
    g_c = dy.float()[inv]
    G = g_c @ w2.float().t()
    g_pre = G * (2 * torch.clamp_min(pre, 0)) * mask
    d_x = (g_pre @ w1.float().t())[torch.from_numpy(perm).to(x.device)]
    counts = (act != 0).sum(dim=0)
    sp, de = plan_lists(counts, 0.95)
    sp_t, de_t = torch.from_numpy(sp).to(x.device), torch.from_numpy(de).to(x.device)
    d_w2 = torch.empty(h, w2.shape[1], device=x.device)
    d_w1t = torch.empty(h, w1.shape[0], device=x.device)
    ka = kept if act_store is None else act_store.float()
    kg = g_pre if g_store is None else g_store.float()
    d_w2[sp_t] = feature_top2(ka[:, sp_t]).t() @ g_c
    d_w2[de_t] = ka[:, de_t].t() @ g_c
    d_w1t[sp_t] = feature_top2(kg[:, sp_t]).t() @ x_in
    d_w1t[de_t] = kg[:, de_t].t() @ x_in
    return dict(pre=pre, act=act, mask=mask, out=out, d_x=d_x, d_w1=d_w1t.t(), d_w2=d_w2, counts=counts, sp=sp)


@pytest.fixture(autouse=True)
def no_tf32():
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32 = old


def test_torch_restatement_matches_oracle_small():
    n, d, h = 256, 64, 256
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.85, seed=5)
    perm = O.make_permutation(0, n)
    t = [torch.from_numpy(v).cuda() for v in (x, w1, w2, dy)]
    o_out, o_cache = O.ffn_forward(x, w1, w2, O.RECIPE, ordered=False)
    o_g = O.ffn_backward(dy, o_cache, w1, w2, O.RECIPE, ordered=False)
    # the rank rule on the oracle's own activation reproduces its mask
    o_act = torch.clamp_min(torch.from_numpy(o_cache["pre"]).cuda(), 0) ** 2
    assert torch.equal(top2_mask(o_act.reshape(n, h // 4, 4)).reshape(n, h).cpu(), torch.from_numpy(o_cache["mask"]))
    r = torch_recipe(*t, perm, mask_dev=torch.from_numpy(o_cache["mask"]).cuda())
    assert rel(r["out"].cpu(), torch.from_numpy(o_out)) < 1e-5
    for k in ("d_x", "d_w1", "d_w2"):
        assert rel(r[k].cpu(), torch.from_numpy(o_g[k])) < 1e-5, k


def expected_split_rows(stored: torch.Tensor, plan, npad: int):
    """The paired-layout feature-wise operand K4 must produce from the
    device's stored token-wise values (dense [npad, h] image, bf16): rows
    [0, 2 nd) = dense feature r as tokens (4j, 4j+1) / (4j+2, 4j+3) with
    selectors (0, 1) / (2, 3); row 2 nd + s = sparse feature s's top-2 down
    each group of 4 tokens (rank rule, NaN last), values in token order.
    Returns (values bf16 [rows, npad/2], ref metadata uint8 [rows, npad/4, 2])."""
    sp, de = plan.sparse_features.long(), plan.dense_features.long()
    nd = de.numel()
    cols = stored[:, sp].float()                    # [npad, ns]
    g = cols.t().reshape(-1, npad // 4, 4)          # [ns, groups, 4 tokens]
    keep = top2_mask(g)
    idx = torch.sort(torch.where(keep, torch.arange(4, device=g.device), 4), dim=-1).values[..., :2]
    sv = torch.gather(g, 2, idx)                    # [ns, groups, 2]
    dcols = stored[:, de].float().t().reshape(nd, npad // 4, 4)
    rows_v = torch.empty(2 * nd + sp.numel(), npad // 4, 2, device=g.device)
    rows_m = torch.empty(2 * nd + sp.numel(), npad // 4, 2, dtype=torch.uint8, device=g.device)
    rows_v[0:2 * nd:2], rows_v[1:2 * nd:2] = dcols[..., 0:2], dcols[..., 2:4]
    rows_m[0:2 * nd:2] = torch.tensor([0, 1], dtype=torch.uint8, device=g.device)
    rows_m[1:2 * nd:2] = torch.tensor([2, 3], dtype=torch.uint8, device=g.device)
    rows_v[2 * nd:] = sv
    rows_m[2 * nd:] = idx.to(torch.uint8)
    return rows_v.reshape(rows_v.shape[0], npad // 2).bfloat16(), rows_m


def check_split(fs, stored, plan, npad):
    """K4's operand bit for bit (values as raw bf16 bits, metadata through
    the hw -> reference converter)."""
    from paper_2503_16672_b200 import _lib

    want_v, want_m = expected_split_rows(stored, plan, npad)
    rows = want_v.shape[0]
    assert torch.equal(fs.vs[:rows].view(torch.int16), want_v.view(torch.int16))
    rp = (rows + 127) // 128 * 128
    ref = torch.empty(rp, npad // 4, 2, dtype=torch.uint8, device=stored.device)
    _lib.call("s24_meta_hw_to_ref", fs.es.data_ptr(), rp, npad, ref.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert torch.equal(ref[:rows], want_m)
    assert not fs.vs[rows:].view(torch.int16).any()  # zero padding rows


def split_stats(stored, plan):
    """(nonzeros before, after) of sparsify_feature_wise over the sparse
    features (ref splitgemm.py:72-75), from the stored values."""
    cols = stored[:, plan.sparse_features.long()].float()
    g = cols.t().reshape(cols.shape[1], -1, 4)
    return int((g != 0).sum()), int(((g * top2_mask(g)) != 0).sum())


def full_parity(n, d, h, sparsity, seed):
    """Recipe fwd + bwd at a full size against the rank rules (bitwise) on the
    device's own intermediates, and against the fp32 torch restatement
    (tolerance). Returns the error dict."""
    import bench

    x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=seed, device=torch.device("cuda"),
                                                  sparsity=sparsity)
    p = s24.FfnParams(w1=w1, w2=w2)
    out, cache = s24.ffn_forward(x, p, s24.RECIPE, keep_pre_act=True)
    grads = s24.ffn_backward(dy, cache, p, s24.RECIPE)
    torch.cuda.synchronize()
    perm = O.make_permutation(0, n)
    npad = (n + 127) // 128 * 128

    # K1 selection, values, counts, statistics and plan: bitwise on the
    # device's own fp32 pre-activation
    act_dev = torch.clamp_min(cache.pre_act, 0) ** 2
    m_rule = top2_mask(act_dev.reshape(n, h // 4, 4)).reshape(n, h)
    m_dev = cache.fwd_mask
    assert torch.equal(m_dev, m_rule)
    assert bool((m_dev.reshape(n, h // 4, 4).sum(-1) == 2).all())
    vals = cache.act_sparse.values.reshape(n, h // 2)
    assert torch.equal(vals, act_dev[m_dev].reshape(n, h // 2).bfloat16())
    counts = (act_dev != 0).sum(dim=0)
    assert torch.equal(cache.counts.long(), counts)
    nz_after = int((act_dev * m_dev != 0).sum())
    assert cache.stats.nonzeros_before == int(counts.sum()) and cache.stats.nonzeros_after == nz_after
    sp, _ = plan_lists(counts, 0.95)
    assert np.array_equal(cache.plan.sparse_features.cpu().numpy(), sp)
    del act_dev, m_rule

    # K4 of act and of g_pre, for every feature, against the rank rule on the
    # device's stored bf16 act / g_pre; the drop statistics of both splits
    stored_a = torch.zeros(npad, h, dtype=torch.bfloat16, device="cuda")
    stored_a[:n] = s24.decompress(cache.act_sparse, torch.bfloat16)
    check_split(cache.act_split, stored_a, cache.plan, npad)
    b, a_ = split_stats(stored_a[:n], cache.plan)
    assert (grads.stats_act.nonzeros_before, grads.stats_act.nonzeros_after) == (b, a_)
    assert grads.stats_act.total_entries == n * cache.plan.n_sparse
    stored_g = torch.zeros(npad, h, dtype=torch.bfloat16, device="cuda")
    stored_g[:n] = s24.decompress(grads.g_pre_sparse, torch.bfloat16)
    # g_pre lives on the forward keep pattern (exact by construction)
    assert not bool(stored_g[:n][~m_dev].float().any())
    check_split(grads.g_split, stored_g, cache.plan, npad)
    b, a_ = split_stats(stored_g[:n], cache.plan)
    assert (grads.stats_grad.nonzeros_before, grads.stats_grad.nonzeros_after) == (b, a_)

    # outputs and gradients vs the fp32 torch restatement on the same inputs
    # (its own fp32 GEMM for the pre-activation; the device's token mask and,
    # for the feature-wise splits, its stored act / g_pre are used downstream,
    # so that flips from accumulation order or bf16 storage are not counted as
    # arithmetic error -- the selections are checked bitwise above)
    r = torch_recipe(x, w1, w2, dy, perm, mask_dev=m_dev, act_store=stored_a[:n], g_store=stored_g[:n])
    del stored_a, stored_g
    flips = int((top2_mask(r["act"].reshape(n, h // 4, 4)).reshape(n, h) != m_dev).sum())
    errs = {"out": rel(out.float(), r["out"]), "d_x": rel(grads.d_x.float(), r["d_x"]),
            "d_w1": rel(grads.d_w1, r["d_w1"]), "d_w2": rel(grads.d_w2, r["d_w2"])}
    print(f"[reported] ({n}, {d}, {h}) s={sparsity} recipe vs fp32 torch:", {k: f"{v:.2e}" for k, v in errs.items()},
          "mask flips", flips, "dropped", cache.stats.dropped, "feature-wise dropped", grads.stats_act.dropped,
          grads.stats_grad.dropped)
    assert flips <= 1e-4 * n * h, flips
    assert errs["out"] < 1e-2 and errs["d_x"] < 1e-2
    assert errs["d_w1"] < 8e-3 and errs["d_w2"] < 8e-3
    assert math.isfinite(sum(errs.values()))
    return errs


def test_recipe_at_c2_size():
    import bench

    full_parity(*bench.CONFIGS["c2"], sparsity=0.9, seed=7)


@pytest.mark.parametrize("sparsity", [0.9, 0.5, 0.98])
def test_recipe_at_7b_class_size(sparsity):
    """BASELINE configs[3] (c4: the 7B-class FFN, 32768 tokens, fwd + bwd)
    at its 0.9 activation sparsity, and configs[4]'s (c5) sweep extremes
    0.5 and 0.98 at the same shape."""
    import bench

    full_parity(*bench.CONFIGS["c4"], sparsity=sparsity, seed=11)


def test_prefill_at_7b_class_size():
    """BASELINE configs[2] (c3: the 7B-class FFN forward, inference prefill):
    the forward without the permutation / plan / split (for_backward=False)
    returns the bits of the training forward, and its selection, values,
    counts and statistics follow the rank rule on its own pre-activation."""
    import bench

    n, d, h = bench.CONFIGS["c3"]
    x, w1, w2, _ = bench.synthetic_device_inputs(torch, n, d, h, seed=13, device=torch.device("cuda"))
    p = s24.FfnParams(w1=w1, w2=w2)
    out_inf, c_inf = s24.ffn_forward(x, p, s24.RECIPE, for_backward=False, keep_pre_act=True)
    out_tr, c_tr = s24.ffn_forward(x, p, s24.RECIPE)
    torch.cuda.synchronize()
    assert torch.equal(out_inf, out_tr)
    assert c_inf.perm is None and c_inf.act_split is None
    act = torch.clamp_min(c_inf.pre_act, 0) ** 2
    m_rule = top2_mask(act.reshape(n, h // 4, 4)).reshape(n, h)
    assert torch.equal(c_inf.fwd_mask, m_rule)
    assert torch.equal(c_inf.act_sparse.values.reshape(n, h // 2), act[m_rule].reshape(n, h // 2).bfloat16())
    counts = (act != 0).sum(dim=0)
    assert torch.equal(c_inf.counts.long(), counts) and torch.equal(c_tr.counts, c_inf.counts)
    assert c_inf.stats.nonzeros_after == int((act * m_rule != 0).sum())
