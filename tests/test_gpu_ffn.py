"""End-to-end parity of the drop-in FFN (ffn_forward / ffn_backward) on the GPU
against the numpy oracle (oracle/srelu24_np.py, itself pinned to the
reference by tests/test_oracle_golden.py).

Bit-exact: permutation, keep masks / metadata, per-feature counts, split plan
and every drop count, all evaluated on identical inputs (the GPU's own fp32
pre-activation, or its own stored bf16 values for the feature-wise splits).
Tolerance (relative Frobenius norm, stated per output): out / d_x are bf16
outputs that pass through 2-3 bf16 roundings (act or g_pre, then the output),
each <= 2^-9 relative, so we allow TOL_BF16 = 1e-2; the fp32 weight gradients
see one bf16 rounding of act / g_pre, TOL_F32 = 8e-3. Mask flips caused by
fp32 accumulation-order differences in Y1 are counted and must stay below
1e-4 of the groups.
"""

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2
TOL_F32 = 8e-3


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def cfg_dict(cfg):
    return dict(forward_mode=cfg.forward_mode, backward_mode=cfg.backward_mode,
                mask_grad_with_fwd=cfg.mask_grad_with_fwd, permute_tokens=cfg.permute_tokens,
                permute_seed=cfg.permute_seed, split_ratio=cfg.split_ratio)


def run_gpu(x, w1, w2, dy, cfg, keep_pre=True):
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, cfg, keep_pre_act=keep_pre)
    grads = s24.ffn_backward(torch.from_numpy(dy).cuda(), cache, p, cfg)
    torch.cuda.synchronize()
    return out, cache, grads


@pytest.mark.parametrize("n,d,h", [(4096, 512, 2048), (1024, 256, 512), (200, 128, 256)])
def test_recipe_selection_exact_and_outputs_within_tolerance(n, d, h):
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=0)
    cfg = s24.RECIPE
    out, cache, grads = run_gpu(x, w1, w2, dy, cfg)

    # permutation (host PCG64 Fisher-Yates, same stream as the reference)
    perm = O.make_permutation(0, n)
    assert np.array_equal(cache.perm.cpu().numpy(), perm)

    # selection replayed on the GPU's own fp32 pre-activation: bit-exact
    pre = cache.pre_act.cpu().numpy()
    r = np.maximum(pre, np.float32(0))
    act = r * r
    ov, om, omask, ost = O.sparsify_token(act)
    assert np.array_equal(cache.act_sparse.meta.cpu().numpy(), om)
    assert np.array_equal(cache.act_sparse.values.float().cpu().numpy(), O.bf16_round(ov))
    assert np.array_equal(cache.counts.cpu().numpy(), O.column_counts(act))
    assert cache.stats.nonzeros_before == ost["nonzeros_before"]
    assert cache.stats.dropped == ost["dropped"]
    osp, ode = O.partition(O.column_counts(act), cfg.split_ratio)
    assert np.array_equal(cache.plan.sparse_features.cpu().numpy(), osp)
    assert np.array_equal(cache.plan.dense_features.cpu().numpy(), ode)

    # feature-wise drop counts of both weight-gradient splits, replayed on the
    # GPU's stored (bf16) act and g_pre values
    act_kept = s24.decompress(cache.act_sparse).cpu().numpy()
    _, _, _, fst = O.sparsify_feature(np.ascontiguousarray(act_kept[:, osp]))
    assert grads.stats_act.total_entries == fst["total_entries"]
    assert grads.stats_act.nonzeros_before == fst["nonzeros_before"]
    assert grads.stats_act.dropped == fst["dropped"]
    # ... and of g_pre (the split of dW1), on the device's own stored g_pre
    g_kept = s24.decompress(grads.g_pre_sparse).cpu().numpy()
    _, _, _, gst = O.sparsify_feature(np.ascontiguousarray(g_kept[:, osp]))
    assert grads.stats_grad.total_entries == gst["total_entries"]
    assert grads.stats_grad.nonzeros_before == gst["nonzeros_before"]
    assert grads.stats_grad.dropped == gst["dropped"]

    # end-to-end vs the oracle run independently on the same (bf16-rounded) inputs
    o_out, o_cache = O.ffn_forward(x, w1, w2, cfg_dict(cfg), ordered=False)
    o_g = O.ffn_backward(dy, o_cache, w1, w2, cfg_dict(cfg), ordered=False)
    flips = int((o_cache["mask"] != omask).sum()) // 2
    assert flips <= max(1, n * h // 4 // 10000), f"{flips} mask flips"
    assert rel(out.float().cpu(), o_out) < TOL_BF16
    assert rel(grads.d_x.float().cpu(), o_g["d_x"]) < TOL_BF16
    assert rel(grads.d_w2.cpu(), o_g["d_w2"]) < TOL_F32
    assert rel(grads.d_w1.cpu(), o_g["d_w1"]) < TOL_F32
    assert [e.sparse for e in cache.census + grads.census] == [False, True, False, True, True, True]


def test_dense_mode_matches_oracle():
    n, d, h = 1024, 256, 1024
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.7, seed=3)
    cfg = s24.FfnConfig()
    out, cache, grads = run_gpu(x, w1, w2, dy, cfg)
    o_out, o_cache = O.ffn_forward(x, w1, w2, cfg_dict(cfg), ordered=False)
    o_g = O.ffn_backward(dy, o_cache, w1, w2, cfg_dict(cfg), ordered=False)
    assert rel(out.float().cpu(), o_out) < TOL_BF16
    assert rel(grads.d_x.float().cpu(), o_g["d_x"]) < TOL_BF16
    assert rel(grads.d_w2.cpu(), o_g["d_w2"]) < TOL_F32
    assert rel(grads.d_w1.cpu(), o_g["d_w1"]) < TOL_F32
    assert [e.sparse for e in cache.census + grads.census] == [False] * 6


@pytest.mark.parametrize("cfg", [
    s24.FfnConfig(forward_mode="sparse24"),
    s24.FfnConfig(forward_mode="sparse24", mask_grad_with_fwd=True),
    s24.FfnConfig(forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True),
    s24.FfnConfig(forward_mode="sparse24", backward_mode="naive_sparse"),
    s24.FfnConfig(forward_mode="sparse24", backward_mode="split_masked"),
    s24.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
                  split_ratio=0.5, permute_tokens=True, permute_seed=7),
])
def test_ablation_configs_match_oracle(cfg):
    n, d, h = 512, 256, 512
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.85, seed=5)
    out, cache, grads = run_gpu(x, w1, w2, dy, cfg)
    o_out, o_cache = O.ffn_forward(x, w1, w2, cfg_dict(cfg), ordered=False)
    o_g = O.ffn_backward(dy, o_cache, w1, w2, cfg_dict(cfg), ordered=False)
    assert rel(out.float().cpu(), o_out) < TOL_BF16
    assert rel(grads.d_x.float().cpu(), o_g["d_x"]) < TOL_BF16
    assert rel(grads.d_w2.cpu(), o_g["d_w2"]) < TOL_F32
    assert rel(grads.d_w1.cpu(), o_g["d_w1"]) < TOL_F32


def striped(n, d, seed):
    """pre-activation with one positive per group of 4 in both orientations
    (ref tests/test_ffn.py:117-124): nothing can ever be dropped."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = -np.abs(rng.standard_normal((n, d))).astype(np.float32) - 0.5
    for i in range(n):
        x[i, 4 * np.arange(d // 4) + (i % 4)] = np.abs(rng.standard_normal(d // 4)) + 0.5
    return O.bf16_round(x)


def test_no_drop_recipe_equals_dense_twin():
    n, d = 512, 128
    x = striped(n, d, 1)
    w1 = np.eye(d, dtype=np.float32)
    rng = np.random.Generator(np.random.PCG64(2))
    w2 = O.bf16_round(rng.standard_normal((d, d)).astype(np.float32))
    dy = O.bf16_round(rng.standard_normal((n, d)).astype(np.float32))
    cfg = s24.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True)
    out_s, cache, g_s = run_gpu(x, w1, w2, dy, cfg)
    assert cache.stats.dropped == 0
    assert g_s.stats_act.dropped == 0 and g_s.stats_grad.dropped == 0
    out_d, _, g_d = run_gpu(x, w1, w2, dy, s24.FfnConfig())
    assert rel(out_s.float().cpu(), out_d.float().cpu()) < 1e-2
    assert rel(g_s.d_w1.cpu(), g_d.d_w1.cpu()) < 1e-2
    assert rel(g_s.d_w2.cpu(), g_d.d_w2.cpu()) < 1e-2
    assert rel(g_s.d_x.float().cpu(), g_d.d_x.float().cpu()) < 1e-2


def test_zero_upstream_gradient_gives_zero_grads():
    n, d, h = 256, 128, 256
    x, w1, w2, _ = O.synthetic_ffn_inputs(n, d, h, seed=9)
    out, cache, grads = run_gpu(x, w1, w2, np.zeros((n, d), np.float32), s24.RECIPE)
    assert not grads.d_w1.any() and not grads.d_w2.any() and not grads.d_x.float().any()


def test_state_and_dimension_errors():
    n, d, h = 256, 128, 256
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, seed=4)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, s24.RECIPE)
    with pytest.raises(s24.StateError):
        s24.ffn_backward(torch.from_numpy(dy).cuda(), cache, p, s24.FfnConfig())
    with pytest.raises(s24.StateError):
        s24.ffn_backward(torch.zeros(n + 4, d).cuda(), cache, p, s24.RECIPE)
    with pytest.raises(s24.DimensionError):
        s24.ffn_forward(torch.zeros(6, d).cuda(), p, s24.RECIPE)


def test_sparse_api_functions_match_oracle():
    rng = np.random.Generator(np.random.PCG64(11))
    a = O.bf16_round(((rng.random((256, 384)) < 0.35) * rng.standard_normal((256, 384))).astype(np.float32))
    b = O.bf16_round(rng.standard_normal((384, 64)).astype(np.float32))
    s, mask, st = s24.sparsify_token_wise(a)
    ov, om, omask, ost = O.sparsify_token(a)
    assert np.array_equal(s.meta.cpu().numpy(), om)
    assert np.array_equal(mask.cpu().numpy(), omask)
    assert st.dropped == ost["dropped"]
    kept = O.decompress_token(ov, om, *a.shape)
    assert np.array_equal(s24.decompress(s).cpu().numpy(), kept)
    assert rel(s24.sp_gemm(s, b).cpu(), kept @ b) < 1e-5
    # feature-wise, then the transposed sparse GEMM
    bt = O.bf16_round(rng.standard_normal((256, 64)).astype(np.float32))
    f, fmask, fst = s24.sparsify_feature_wise(a)
    fv, fm, fmask_o, fst_o = O.sparsify_feature(a)
    assert np.array_equal(f.meta.cpu().numpy(), fm)
    assert fst.dropped == fst_o["dropped"]
    fk = O.decompress_feature(fv, fm, *a.shape)
    assert rel(s24.sp_gemm_t(f, bt).cpu(), fk.T @ bt) < 1e-5
    # exact mask compression and its error
    c = s24.compress_token_wise_with_mask(torch.from_numpy(kept).cuda(), mask)
    assert np.array_equal(s24.decompress(c).cpu().numpy(), kept)
    bad = mask.clone()
    bad[0, 0] = ~bad[0, 0]
    with pytest.raises(s24.MaskError):
        s24.compress_token_wise_with_mask(torch.from_numpy(kept).cuda(), bad)
    with pytest.raises(s24.OrientationError):
        s24.sp_gemm(f, b)
    # split GEMM composite oracle (ref tests/test_splitgemm.py:91-97)
    counts = s24.column_nonzero_counts(a)
    plan = s24.partition_features(counts, 0.75)
    osp, ode = O.partition(O.column_counts(a), 0.75)
    assert np.array_equal(plan.sparse_features.cpu().numpy(), osp)
    out = s24.split_gemm_t(a, mask, bt, plan)
    ref, _ = O.split_gemm_t(a, omask, bt, osp, ode, ordered=False)
    assert rel(out.cpu(), ref) < 1e-5


@pytest.mark.parametrize("dense", [False, True])
def test_graph_replay_equals_eager(dense):
    """FfnStepGraph (the whole fwd+bwd captured as one CUDA graph, side-stream
    fork/join included) reproduces the eager step bit for bit, and picks up
    new inputs written into its static buffers."""
    n, d, h = 512, 256, 512
    cfg = s24.FfnConfig() if dense else s24.RECIPE
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=21)
    x2, _, _, dy2 = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=22)
    p = s24.FfnParams(w1=w1, w2=w2)
    g = s24.FfnStepGraph(p, cfg, n)
    for xx, gg in ((x, dy), (x2, dy2)):
        tx, tg = torch.from_numpy(xx).cuda().bfloat16(), torch.from_numpy(gg).cuda().bfloat16()
        out, cache = s24.ffn_forward(tx, p, cfg)
        gr = s24.ffn_backward(tg, cache, p, cfg)
        g.x.copy_(tx)
        g.dy.copy_(tg)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(g.out, out)
        assert torch.equal(g.d_x, gr.d_x) and torch.equal(g.d_w1, gr.d_w1) and torch.equal(g.d_w2, gr.d_w2)


def test_nn_module_autograd_matches_api():
    """SquaredReluFFN24 (autograd.Function over ffn_forward/ffn_backward) gives
    the drop-in API's outputs and gradients; odd token counts are padded."""
    from paper_2503_16672_b200.nn import SquaredReluFFN24

    torch.manual_seed(5)
    d, h = 256, 512
    m = SquaredReluFFN24(d, h)
    x = torch.randn(3, 341, d, device="cuda").bfloat16().requires_grad_(True)  # 1023 tokens
    y = m(x)
    g = torch.randn_like(y)
    (y.float() * g.float()).sum().backward()
    # the same through the API on the padded batch
    xf = torch.cat([x.detach().reshape(-1, d), x.new_zeros(1, d)])
    gf = torch.cat([g.reshape(-1, d), g.new_zeros(1, d)])
    p = s24.FfnParams(w1=m.w1.detach(), w2=m.w2.detach())
    out, cache = s24.ffn_forward(xf, p, s24.RECIPE)
    gr = s24.ffn_backward(gf, cache, p, s24.RECIPE)
    assert torch.equal(y.reshape(-1, d), out[:1023])
    assert torch.equal(x.grad.reshape(-1, d), gr.d_x[:1023])
    assert torch.equal(m.w1.grad, gr.d_w1) and torch.equal(m.w2.grad, gr.d_w2)
    assert m.w1.grad.dtype == torch.float32


def test_grad_ready_order_is_bitwise_identical():
    """With a grad_ready hook (data parallel) the backward runs dW2 right
    after K3 and dW1 after dX, in two launches; without one, both weight
    gradients run in one grouped launch after dX. Same bits, same census, and
    the hook sees d_w2 then d_w1 with their final values."""
    n, d, h = 1024, 256, 1024
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.85, seed=77)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    tx, tg = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
    out, cache = s24.ffn_forward(tx, p, s24.RECIPE)
    g0 = s24.ffn_backward(tg, cache, p, s24.RECIPE)
    seen = []
    out1, cache = s24.ffn_forward(tx, p, s24.RECIPE)
    g1 = s24.ffn_backward(tg, cache, p, s24.RECIPE, grad_ready=lambda name, t: seen.append((name, t.clone())))
    torch.cuda.synchronize()
    assert torch.equal(out, out1)
    for t in ("d_w1", "d_w2", "d_x"):
        assert torch.equal(getattr(g0, t), getattr(g1, t)), t
    assert [e.name for e in g0.census] == [e.name for e in g1.census]
    assert [nm for nm, _ in seen] == ["d_w2", "d_w1"]
    assert torch.equal(seen[0][1], g0.d_w2) and torch.equal(seen[1][1], g0.d_w1)


@pytest.mark.parametrize("fp8", [False, True])
def test_public_side_stream_outputs_are_safe_to_read(fp8):
    """The plan and x_in are produced on the side stream; reading them from
    the cache right after ffn_forward (no synchronize, no backward) must see
    the finished values (the properties make the caller's stream wait)."""
    from dataclasses import replace

    n, d, h = 4096, 512, 2048
    cfg = replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True) if fp8 else s24.RECIPE
    x, w1, w2, _ = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=5)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    tx = torch.from_numpy(x).cuda()
    ref_out, ref_cache = s24.ffn_forward(tx, p, cfg)
    torch.cuda.synchronize()
    want_sp = ref_cache.plan.sparse_features.cpu()
    want_x = ref_cache.x_in.cpu()
    for _ in range(3):
        out, cache = s24.ffn_forward(tx, p, cfg)
        assert torch.equal(cache.plan.sparse_features.cpu(), want_sp)
        assert torch.equal(cache.x_in.cpu(), want_x)


@pytest.mark.parametrize("fp8", [False, True])
def test_grad_bucket_views_are_bitwise_identical(fp8):
    """ffn_backward(grad_bucket=...) writes dW1 / dW2 as views of one flat
    buffer (one all-reduce for both in the data-parallel step), same bits;
    FfnStepGraph(grad_bucket=True) exposes it as .bucket."""
    from dataclasses import replace

    n, d, h = 512, 256, 512
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.85, seed=79)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    cfg = replace(s24.RECIPE, fp8_emulation=fp8, fp8_backward=fp8)
    tx, tg = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
    out, cache = s24.ffn_forward(tx, p, cfg)
    g0 = s24.ffn_backward(tg, cache, p, cfg)
    bucket = torch.empty(2 * d * h, device="cuda")
    out, cache = s24.ffn_forward(tx, p, cfg)
    g1 = s24.ffn_backward(tg, cache, p, cfg, grad_bucket=bucket)
    torch.cuda.synchronize()
    assert torch.equal(g0.d_w1, g1.d_w1) and torch.equal(g0.d_w2, g1.d_w2)
    assert g1.d_w1.data_ptr() == bucket.data_ptr() and torch.equal(bucket[d * h:].view(h, d), g1.d_w2)
    step = s24.FfnStepGraph(p, cfg, n, grad_bucket=True)
    step.x.copy_(tx.bfloat16())
    step.dy.copy_(tg.bfloat16())
    step.replay()
    torch.cuda.synchronize()
    assert step.d_w1.data_ptr() == step.bucket.data_ptr()
    assert torch.equal(step.d_w1, g0.d_w1) and torch.equal(step.d_w2, g0.d_w2)
    with pytest.raises(s24.DimensionError):
        s24.ffn_backward(tg, s24.ffn_forward(tx, p, cfg)[1], p, cfg, grad_bucket=torch.empty(7, device="cuda"))


@pytest.mark.parametrize("fp8", [False, True])
def test_inference_forward_skips_permutation_same_bits(fp8):
    """for_backward=False runs the forward without the token permutation
    (no gathers, no row map): the output is bit-identical to the training
    forward's, and so are the counts, plan and drop statistics."""
    from dataclasses import replace

    n, d, h = 640, 256, 512
    x, w1, w2, _ = O.synthetic_ffn_inputs(n, d, h, sparsity=0.85, seed=80)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    cfg = replace(s24.RECIPE, fp8_emulation=fp8)
    tx = torch.from_numpy(x).cuda()
    o_train, c_train = s24.ffn_forward(tx, p, cfg)
    o_inf, c_inf = s24.ffn_forward(tx, p, cfg, for_backward=False)
    torch.cuda.synchronize()
    assert torch.equal(o_train, o_inf)
    assert torch.equal(c_train.counts, c_inf.counts)
    assert c_train.stats.dropped == c_inf.stats.dropped
    assert torch.equal(c_train.plan.sparse_features, c_inf.plan.sparse_features)
    assert c_inf.perm is None and c_train.perm is not None


@pytest.mark.parametrize("fp8", [False, True])
def test_minimum_and_degenerate_shapes(fp8):
    """n = 4 tokens (one 2:4 group per feature column), h = 128 and d = 32,
    the smallest dims the path takes, and an all-zero input (every group padded with
    zeros, all counts 0, the plan is the first ceil(0.95 h) features by
    index), against the oracle."""
    from dataclasses import replace

    d = 32
    cfg = replace(s24.RECIPE, fp8_emulation=fp8, fp8_backward=fp8)
    ocfg = dict(O.RECIPE, fp8_emulation=fp8, fp8_backward=fp8)
    for n, zero in ((4, False), (8, True)):
        x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, 128, sparsity=0.6, seed=n)
        if zero:
            x = np.zeros_like(x)
        p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
        out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, cfg)
        g = s24.ffn_backward(torch.from_numpy(dy).cuda(), cache, p, cfg)
        torch.cuda.synchronize()
        o_out, o_cache = O.ffn_forward(x, w1, w2, ocfg, ordered=False)
        o_g = O.ffn_backward(dy, o_cache, w1, w2, ocfg, ordered=False)
        assert np.array_equal(cache.fwd_mask.cpu().numpy(), o_cache["mask"])
        assert np.array_equal(cache.plan.sparse_features.cpu().numpy(), o_cache["plan"][0])
        if zero:
            assert not out.float().any() and not g.d_w1.any() and not g.d_w2.any()
            assert cache.stats.nonzeros_before == 0 and cache.stats.dropped == 0
            continue
        tol = 3e-2 if fp8 else 1e-2
        for got, want in ((out.float(), o_out), (g.d_x.float(), o_g["d_x"]), (g.d_w1, o_g["d_w1"]),
                          (g.d_w2, o_g["d_w2"])):
            got = got.cpu().numpy().astype(np.float64)
            assert np.linalg.norm(got - want) <= tol * max(np.linalg.norm(want), 1e-30)


@pytest.mark.parametrize("fp8", [False, True])
def test_prefill_graph_capture(fp8):
    """The inference forward (for_backward=False) joins its side-stream work
    (plan) before returning, so it captures as a CUDA graph (the c3 prefill
    bench) and replays to the eager output, bit for bit."""
    from dataclasses import replace

    n, d, h = 640, 256, 512
    x, w1, w2, _ = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=82)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    cfg = replace(s24.RECIPE, fp8_emulation=fp8)
    tx = torch.from_numpy(x).cuda().bfloat16()
    want, _ = s24.ffn_forward(tx, p, cfg, for_backward=False)
    step = s24.FfnStepGraph(p, cfg, n, backward=False)
    step.x.copy_(tx)
    step.replay()
    torch.cuda.synchronize()
    assert torch.equal(step.out, want)
