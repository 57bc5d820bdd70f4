"""The fp8 FFN configurations (FfnConfig.fp8_emulation / fp8_backward) on the
device vs the oracle's restatement of the reference's e4m3 emulation, and the
reference-facing fp8 API (ref matcore.py:113-261, ffn.py:206-451,
tests/test_ffn.py:322-367, tests/test_acceptance.py:272-291).

The device runs the FFN in bf16 activations with e4m3 tensor-core GEMMs; the
oracle runs the reference's float32 emulation on the same bf16-valued inputs.
Metadata / masks / counts / plans are compared bitwise; outputs and gradients
within the tolerances stated per test, each well below the fp8-vs-unquantized
gap (so the device provably follows the fp8 emulation, not the bf16 path).
"""

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def inputs(n, d, h, seed):
    x, w1, w2, g = O.synthetic_ffn_inputs(n, d, h, sparsity=0.6, seed=seed)
    return x, w1, w2, g


def npy(t):
    return t.float().cpu().numpy()


RECIPE = dict(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True, permute_tokens=True)
CASES = {
    "recipe_f8fwd": dict(RECIPE, fp8_emulation=True),
    "recipe_f8all": dict(RECIPE, fp8_emulation=True, fp8_backward=True),
    "naive_f8all": dict(forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True,
                        fp8_emulation=True, fp8_backward=True),
    "split_nomask_f8all": dict(forward_mode="sparse24", backward_mode="split_masked", fp8_emulation=True,
                               fp8_backward=True),
    "sparse_dense_bwd_f8all": dict(forward_mode="sparse24", fp8_emulation=True, fp8_backward=True),
    "dense_f8all": dict(fp8_emulation=True, fp8_backward=True),
    "dense_f8fwd": dict(fp8_emulation=True),
}


@pytest.mark.parametrize("n,d,h", [(256, 64, 256), (200, 96, 384)])
@pytest.mark.parametrize("name", sorted(CASES))
def test_fp8_ffn_matches_emulation(name, n, d, h):
    kw = CASES[name]
    x, w1, w2, g = inputs(n, d, h, seed=n + h)
    cfg = s24.FfnConfig(**kw)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, cfg)
    grads = s24.ffn_backward(torch.from_numpy(g).cuda(), cache, p, cfg)
    torch.cuda.synchronize()

    ocfg = dict(O.DENSE, **kw)
    o_out, o_cache = O.ffn_forward(x, w1, w2, ocfg, ordered=False)
    o_g = O.ffn_backward(g, o_cache, w1, w2, ocfg, ordered=False)
    # the unquantized run on the same inputs: the fp8 effect the device must reproduce
    bcfg = dict(ocfg, fp8_emulation=False, fp8_backward=False)
    b_out, b_cache = O.ffn_forward(x, w1, w2, bcfg, ordered=False)
    b_g = O.ffn_backward(g, b_cache, w1, w2, bcfg, ordered=False)

    gap_out = rel(o_out, b_out)
    err_out = rel(npy(out), o_out)
    assert err_out < 0.02, (err_out, gap_out)
    assert err_out < 0.35 * gap_out, (err_out, gap_out)
    if cfg.forward_mode == "sparse24":
        # selection sees the unquantized fp32 pre-activation: same keep pattern
        mask = cache.fwd_mask.cpu().numpy()
        agree = (mask == o_cache["mask"]).mean()
        assert agree > 0.999, agree
        # the cached activation is the dequantized one (ref ffn.py:335-340)
        vals = cache.act_sparse.values.float().cpu().numpy()
        assert rel(vals, o_cache["vals"]) < 0.01
    tol_g = 0.03 if cfg.fp8_backward else 0.02
    report = [f"out {err_out:.1e}/{gap_out:.1e}"]
    for t in ("d_w1", "d_w2", "d_x"):
        got, want, base = npy(getattr(grads, t)), o_g[t], b_g[t]
        err, gap = rel(got, want), rel(want, base)
        report.append(f"{t} {err:.1e}/{gap:.1e}")
        assert err < tol_g, (t, err, gap)
        assert err < 0.5 * gap, (t, err, gap)
    print(f"[reported] {name} n={n}: err vs fp8 emulation / fp8 gap: " + ", ".join(report))


def test_fp8_selects_before_quantizing():
    # ref tests/test_ffn.py:360-367 on a device-sized FFN: W1 = W2 = identity
    # on the first 4 dims, 3.01 / 3.0 / 2.99 share one e4m3 code
    d, h, n = 32, 128, 4
    w = np.zeros((d, h), np.float32)
    w[:4, :4] = np.eye(4)
    x = np.zeros((n, d), np.float32)
    x[:, :4] = [3.01, 3.0, 2.99, -1.0]
    p = s24.FfnParams(w1=torch.from_numpy(w).cuda(), w2=torch.from_numpy(w.T.copy()).cuda())
    _, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, s24.FfnConfig(forward_mode="sparse24",
                                                                             fp8_emulation=True))
    meta = cache.act_sparse.meta.cpu().numpy()
    assert np.array_equal(meta[0, 0], [0, 1])


def test_fp8_api_matches_reference():
    r = np.random.default_rng(109)
    a = r.uniform(-1, 1, (32, 48)).astype(np.float32)
    b = r.uniform(-1, 1, (48, 32)).astype(np.float32)
    qa = s24.fp8_quantize_rowwise(a, "rows")
    qb = s24.fp8_quantize_rowwise(b, "cols")
    ca, sa = O.quantize(a, "rows")
    cb, sb = O.quantize(b, "cols")
    assert np.array_equal(qa.codes.cpu().numpy(), ca) and np.array_equal(qa.scales.cpu().numpy(), sa)
    assert np.array_equal(qb.codes.cpu().numpy(), cb) and np.array_equal(qb.scales.cpu().numpy(), sb)
    out = s24.fp8_gemm_rowwise(qa, qb).cpu().numpy()
    want = O.mm_f8(a, b)
    assert rel(out, want) < 1e-6
    assert rel(out, a.astype(np.float64) @ b) <= 0.06  # ref tests/test_acceptance.py:283-291
    deq = s24.fp8_dequantize(qa).cpu().numpy()
    assert np.array_equal(deq, O._E4M3_F32[ca] * sa[:, None])
    codes = np.arange(256)
    ok = ~np.isnan(O._E4M3[codes])
    assert np.array_equal(s24.e4m3_encode(O._E4M3[codes][ok]).cpu().numpy(), codes[ok].astype(np.uint8))
    dec = s24.e4m3_decode(torch.arange(256)).cpu().numpy()
    assert np.array_equal(np.isnan(dec), np.isnan(O._E4M3))
    assert np.array_equal(dec[ok], O._E4M3_F32[ok])
    with pytest.raises(s24.NonFiniteError):
        s24.e4m3_encode([1.0, float("nan")])
    with pytest.raises(s24.OrientationError):
        s24.fp8_gemm_rowwise(qb, qa)


def test_fp8_shape_errors_and_module():
    """A model dim the e4m3 GEMMs do not tile (40) runs zero-padded; the
    nn.Module and the graph capture run the e4m3 configs like the bf16 ones."""
    from dataclasses import replace

    cfg = replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True)
    x = torch.randn(64, 40, device="cuda")
    p = s24.FfnParams(w1=torch.randn(40, 128, device="cuda"), w2=torch.randn(128, 40, device="cuda"))
    out40, c40 = s24.ffn_forward(x, p, cfg)
    g40 = s24.ffn_backward(x, c40, p, cfg)
    assert out40.shape == (64, 40) and g40.d_w1.shape == (40, 128) and g40.d_x.shape == (64, 40)
    with pytest.raises(s24.DimensionError):
        s24.ffn_forward(torch.randn(64, 48, device="cuda"), p, cfg)
    torch.manual_seed(0)
    layer = s24.SquaredReluFFN24(64, 256, cfg=cfg)
    xin = torch.randn(2, 50, 64, device="cuda", requires_grad=True)  # 100 tokens: padded to a multiple of 4
    y = layer(xin)
    y.float().pow(2).mean().backward()
    assert y.shape == xin.shape and xin.grad is not None and layer.w1.grad is not None
    assert bool(torch.isfinite(layer.w1.grad).all()) and bool(torch.isfinite(xin.grad).all())
    step = s24.FfnStepGraph(s24.FfnParams(w1=layer.w1.detach(), w2=layer.w2.detach()), cfg, 128)
    xs = torch.randn(128, 64, device="cuda").bfloat16()
    step.x.copy_(xs)
    step.dy.copy_(xs)
    step.replay()
    out_e, cache = s24.ffn_forward(xs, s24.FfnParams(w1=layer.w1.detach(), w2=layer.w2.detach()), cfg)
    g_e = s24.ffn_backward(xs, cache, s24.FfnParams(w1=layer.w1.detach(), w2=layer.w2.detach()), cfg)
    torch.cuda.synchronize()
    assert torch.equal(step.out, out_e) and torch.equal(step.d_w1, g_e.d_w1) and torch.equal(step.d_x, g_e.d_x)
