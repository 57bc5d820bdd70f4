"""e4m3 (fp8) kernels through the C ABI vs the oracle's restatement of the
reference's emulation (ref matcore.py:113-261, ffn.py:206-268).

Bit-exact: codes, scales, dequantized images, metadata (identical fp32 inputs
give identical quotients and the hardware conversion rounds like the
reference). GEMMs: fp32 accumulation of exact e4m3 products, compared with a
float64 evaluation of the same scaled sum at 1e-5 relative Frobenius error.
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import srelu24_np as O
from paper_2503_16672_b200 import _lib

from .test_gpu_kernels import BF16, F32, P, S, gpu_sparsify_token, rel_err

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
E4M3 = torch.tensor(O._E4M3, dtype=torch.float64)


def dec(codes: torch.Tensor) -> torch.Tensor:
    return E4M3.to(codes.device)[codes.long()]


def quant_rows(a, pair_rows=0, amax=None, want_deq=False, want_raw=False):
    rows, cols = a.shape
    codes = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    scales = torch.empty(rows, dtype=torch.float32, device="cuda")
    deq = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda") if want_deq else None
    raw = torch.empty(rows, cols, dtype=torch.bfloat16, device="cuda") if want_raw else None
    dt = F32 if a.dtype == torch.float32 else BF16
    _lib.call("s24_fp8_quant_rows", P(a), dt, rows, cols, a.stride(0), P(amax), pair_rows, P(codes), cols, P(scales),
              P(deq), cols, P(raw), cols, S())
    return codes, scales, deq, raw


def quant_cols_t(a):
    rows, cols = a.shape
    ld = (rows + 15) // 16 * 16
    codes_t = torch.zeros(cols, ld, dtype=torch.uint8, device="cuda")
    scales = torch.empty(cols, dtype=torch.float32, device="cuda")
    ws = torch.empty(cols, dtype=torch.int32, device="cuda")
    dt = F32 if a.dtype == torch.float32 else BF16
    _lib.call("s24_fp8_quant_cols_t", P(a), dt, rows, cols, a.stride(0), P(codes_t), ld, P(scales), P(ws), S())
    return codes_t[:, :rows], scales


def rand_codes(*shape, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    c = torch.randint(0, 256, shape, generator=g, dtype=torch.int32)
    c = torch.where((c & 0x7F) == 0x7F, c ^ 1, c)  # no NaN patterns
    return c.to(torch.uint8).cuda()


def test_encode_matches_reference_codes():
    gold = np.load(GOLD / "fp8.npz")
    x = gold["enc_x"].astype(np.float32)
    x = x[np.isfinite(x)]
    xt = torch.from_numpy(x).cuda()
    codes = torch.empty(x.size, dtype=torch.uint8, device="cuda")
    _lib.call("s24_e4m3_encode", P(xt), x.size, P(codes), S())
    assert np.array_equal(codes.cpu().numpy(), O.e4m3_encode(x))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("rows,cols", [(64, 256), (37, 72), (130, 1024)])
def test_quant_rows_bitwise(dtype, rows, cols):
    torch.manual_seed(rows + cols)
    a = (torch.randn(rows, cols, device="cuda") * torch.logspace(-3, 2, rows, device="cuda")[:, None]).to(dtype)
    a[1] = 0
    a[2, 5] = -0.0
    codes, scales, deq, raw = quant_rows(a, want_deq=True, want_raw=True)
    af = a.float().cpu().numpy()
    rc, rs = O.quantize(af, "rows")
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
    want_deq = O.bf16_round(O._E4M3_F32[rc] * rs[:, None])
    assert np.array_equal(deq.float().cpu().numpy(), want_deq)
    assert torch.equal(raw, a.bfloat16())
    # precomputed row maxima (the K1 path) give the same result
    amax = a.float().abs().amax(dim=1).contiguous().view(torch.int32)
    c2, s2, _, _ = quant_rows(a, amax=amax)
    assert torch.equal(c2, codes) and torch.equal(s2, scales)


def test_quant_rows_pairs_share_scales():
    torch.manual_seed(3)
    a = torch.randn(20, 64, device="cuda").bfloat16()
    a[0] *= 100
    codes, scales, _, _ = quant_rows(a, pair_rows=8)
    af = a.float().cpu().numpy()
    for r in range(0, 8, 2):
        pair = af[r:r + 2]
        s = O.e4m3_scales(np.abs(pair).max())
        assert scales[r].item() == s and scales[r + 1].item() == s
        assert np.array_equal(codes[r:r + 2].cpu().numpy(), O.e4m3_encode(pair / s).reshape(pair.shape))
    rc, rs = O.quantize(af[8:], "rows")
    assert np.array_equal(codes[8:].cpu().numpy(), rc) and np.array_equal(scales[8:].cpu().numpy(), rs)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("rows,cols", [(256, 128), (100, 72), (64, 1000)])
def test_quant_cols_transposed_bitwise(dtype, rows, cols):
    torch.manual_seed(rows * cols)
    a = (torch.randn(rows, cols, device="cuda") * torch.logspace(-2, 3, cols, device="cuda")[None, :]).to(dtype)
    a[:, 3] = 0
    codes_t, scales = quant_cols_t(a)
    rc, rs = O.quantize(a.float().cpu().numpy(), "cols")
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes_t.cpu().numpy(), rc.T)


@pytest.mark.parametrize("M,N,K", [(256, 256, 256), (300, 288, 208), (128, 512, 1024)])
def test_gemm_f8(M, N, K):
    A, B = rand_codes(M, K, seed=1), rand_codes(N, K, seed=2)
    sa = torch.rand(M, device="cuda") + 0.5
    sb = torch.rand(N, device="cuda") + 0.5
    D = torch.empty(M, N, device="cuda")
    _lib.call("s24_gemm_f8", P(A), K, P(B), K, M, N, K, P(sa), P(sb), P(D), F32, N, None, 0, -1, S())
    ref = (sa.double()[:, None] * sb.double()[None, :]) * (dec(A) @ dec(B).t())
    assert rel_err(D, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(256, 256, 512), (384, 320, 384), (128, 256, 2048)])
def test_spmm_f8(M, N, K):
    torch.manual_seed(M + K)
    a = torch.randn(M, K, device="cuda").bfloat16()
    vals, meta_ref, meta_hw, mask, _ = gpu_sparsify_token(a)
    codes, scales, _, _ = quant_rows(vals[:M].contiguous())
    acodes = torch.zeros(vals.shape, dtype=torch.uint8, device="cuda")
    acodes[:M] = codes
    meta8 = torch.empty_like(meta_hw)
    _lib.call("s24_meta_hw_to_f8", P(meta_hw), M, K, P(meta8), S())
    B = rand_codes(N, K, seed=5)
    sb = torch.rand(N, device="cuda") + 0.5
    D = torch.empty(M, N, device="cuda")
    _lib.call("s24_spmm_f8", P(acodes), P(meta8), P(B), K, M, N, K, P(scales), P(sb), P(D), F32, N, None, 0, -1, None,
              0, S())
    kept = O.decompress_token(dec(codes).cpu().numpy().reshape(M, K // 4, 2), meta_ref.cpu().numpy(), M, K)
    ref = (scales.double()[:, None] * sb.double()[None, :]) * (torch.from_numpy(kept).cuda() @ dec(B).t())
    assert rel_err(D, ref) < 1e-5


def test_spmm_f8_pair_rows():
    """Paired rows (a dense feature as two 2:4 rows) sum after scaling."""
    torch.manual_seed(11)
    M, N, K = 256, 256, 512
    a = torch.randn(M, K, device="cuda").bfloat16()
    vals, meta_ref, meta_hw, _, _ = gpu_sparsify_token(a)
    codes, scales, _, _ = quant_rows(vals[:M].contiguous(), pair_rows=64)
    meta8 = torch.empty_like(meta_hw)
    _lib.call("s24_meta_hw_to_f8", P(meta_hw), M, K, P(meta8), S())
    B = rand_codes(N, K, seed=6)
    sb = torch.rand(N, device="cuda") + 0.5
    D = torch.zeros(M, N, device="cuda")
    _lib.call("s24_spmm_f8", P(codes), P(meta8), P(B), K, M, N, K, P(scales), P(sb), P(D), F32, N, None, 0, -1, None,
              64, S())
    kept = torch.from_numpy(O.decompress_token(dec(codes).cpu().numpy().reshape(M, K // 4, 2),
                                               meta_ref.cpu().numpy(), M, K)).cuda()
    full = (scales.double()[:, None] * sb.double()[None, :]) * (kept @ dec(B).t())
    ref = full.clone()
    ref[0:64:2] += full[1:64:2]
    ref[1:64:2] = 0
    assert rel_err(D, ref) < 1e-5


def test_fwd_gemm1_f8_matches_oracle():
    """K1 on e4m3 operands: scaled pre-activation, relu^2, token-wise 2:4 on
    the fp32 values (selection before quantization), per-feature counts."""
    torch.manual_seed(21)
    M, N, K = 256, 512, 256
    x = torch.randn(M, K, device="cuda").bfloat16()
    w1 = (torch.randn(K, N, device="cuda") / 16).bfloat16()
    xq, sx, _, _ = quant_rows(x)
    w1q, s1 = quant_cols_t(w1)  # [N, K]
    vals32 = torch.zeros(M, N // 2, device="cuda")
    amax = torch.zeros(M, dtype=torch.int32, device="cuda")
    meta = torch.full((_lib.meta_hw_bytes(M, N),), 0x44, dtype=torch.uint8, device="cuda")
    counts = torch.zeros(N, dtype=torch.int32, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.empty(M, N, device="cuda")
    _lib.call("s24_fwd_gemm1_f8", P(xq), K, P(w1q.contiguous()), K, M, N, K, P(sx), P(s1), P(vals32), P(amax), P(meta),
              P(counts), P(stats), P(y), S())
    pre_ref = (sx.double()[:, None] * s1.double()[None, :]) * (dec(xq) @ dec(w1q).t())
    assert rel_err(y, pre_ref) < 1e-5
    # selection / counts bit-exact given the device's fp32 pre-activation
    yn = y.cpu().numpy()
    r = np.maximum(yn, 0)
    act = r * r
    v, m, _, _ = O.sparsify_token(act)
    assert np.array_equal(vals32.cpu().numpy().reshape(M, N // 4, 2), v)
    ref_meta = torch.empty(M, N // 4, 2, dtype=torch.uint8, device="cuda")
    _lib.call("s24_meta_hw_to_ref", P(meta), M, N, P(ref_meta), S())
    assert np.array_equal(ref_meta.cpu().numpy(), m)
    assert np.array_equal(counts.cpu().numpy(), O.column_counts(act))
    assert np.array_equal(amax.view(torch.float32).cpu().numpy(), np.abs(v).reshape(M, -1).max(axis=1))


def test_bwd_dact_f8_matches_reference():
    torch.manual_seed(22)
    M, N, K = 256, 512, 256  # N = hidden, K = model dim
    act = torch.rand(M, N, device="cuda").bfloat16()
    vals, meta_ref, meta_hw, mask, _ = gpu_sparsify_token(act)
    g = torch.randn(M, K, device="cuda").bfloat16()
    w2 = (torch.randn(N, K, device="cuda") / 16).bfloat16()
    gq, sg, _, _ = quant_rows(g)
    w2q, s2, _, _ = quant_rows(w2)  # per row of W2 = per column of W2^T
    gvals = torch.zeros_like(vals)
    _lib.call("s24_bwd_dact_f8", P(gq), K, P(w2q), K, M, N, K, P(sg), P(s2), P(vals), P(meta_hw), P(gvals), S())
    G = (sg.double()[:, None] * s2.double()[None, :]) * (dec(gq) @ dec(w2q).t())
    dense_act = act.double() * mask.double()
    gpre = G * 2 * dense_act.sqrt() * mask.double()
    want = torch.from_numpy(O.compress_with_mask(gpre.cpu().numpy(), mask.cpu().numpy().astype(bool))[0]).cuda()
    got = gvals[:M].double().reshape(M, N // 4, 2)
    assert rel_err(got, want) < 1e-2  # bf16 output, sqrt.approx


def test_quant_rows_boundary_stress():
    """The quantizers divide by the shared scale with a reciprocal + one FMA
    residual step (csrc/fp8.cu, Divisor); codes must still equal the IEEE
    quotient's: rows built from exact e4m3 rounding boundaries times the
    scale, +-1..3 ulp around them, and random fills."""
    g = np.random.default_rng(5)
    grid = np.unique(np.abs(O._E4M3[~np.isnan(O._E4M3)]))
    mids = ((grid[1:] + grid[:-1]) / 2).astype(np.float32)
    rows, cols = 512, 1024
    a = np.empty((rows, cols), np.float32)
    for r in range(rows):
        amax = np.float32(g.uniform(0.5, 2.0) * 10.0 ** g.integers(-6, 6))
        s = O.e4m3_scales(amax)
        base = g.choice(mids, cols) * s  # fp32 products: boundary * scale, rounded
        k = g.integers(-3, 4, cols)
        v = np.nextafter(base, np.where(k > 0, np.inf, -np.inf).astype(np.float32))
        for _ in range(2):
            v = np.where(np.abs(k) > 1, np.nextafter(v, np.where(k > 0, np.inf, -np.inf).astype(np.float32)), v)
        v = np.where(k == 0, base, v)
        v = np.where(g.random(cols) < 0.3, g.uniform(-1, 1, cols).astype(np.float32) * amax, v)
        v = v * np.where(g.random(cols) < 0.5, -1, 1).astype(np.float32)
        v[0] = amax
        a[r] = np.clip(v, -amax, amax)
    t = torch.from_numpy(a).cuda()
    codes, scales, _, _ = quant_rows(t)
    rc, rs = O.quantize(a, "rows")
    assert np.array_equal(scales.cpu().numpy(), rs)
    assert np.array_equal(codes.cpu().numpy(), rc)
    ct, cs = quant_cols_t(t.t().contiguous().bfloat16().float().contiguous())
    # (bf16-rounded copy for the column path, checked against its own oracle)
    rc2, rs2 = O.quantize(t.t().contiguous().bfloat16().float().cpu().numpy(), "cols")
    assert np.array_equal(cs.cpu().numpy(), rs2) and np.array_equal(ct.cpu().numpy(), rc2.T)


def test_spmm_pair_f8_matches_two_launches():
    torch.manual_seed(31)
    M, N, K = 384, 256, 512
    ops = []
    for i in range(2):
        a = torch.randn(M, K, device="cuda").bfloat16()
        vals, _, meta_hw, _, _ = gpu_sparsify_token(a)
        codes, scales, _, _ = quant_rows(vals[:M].contiguous(), pair_rows=64)
        meta8 = torch.empty_like(meta_hw)
        _lib.call("s24_meta_hw_to_f8", P(meta_hw), M, K, P(meta8), S())
        ops.append((codes, meta8, scales, rand_codes(N, K, seed=40 + i), torch.rand(N, device="cuda") + 0.5))
    rmap = torch.randperm(M + 16, device="cuda")[:M].int()
    refs = [torch.zeros(M + 16, N, device="cuda"), torch.zeros(N, M + 16, device="cuda")]
    for (c, e, sa, b, sb), ref, tr in zip(ops, refs, (0, 1)):
        _lib.call("s24_spmm_f8", P(c), P(e), P(b), K, M, N, K, P(sa), P(sb), P(ref), F32, ref.shape[1], P(rmap), tr,
                  -1, None, 64, S())
    outs = [torch.zeros_like(refs[0]), torch.zeros_like(refs[1])]
    (c0, e0, sa0, b0, sb0), (c1, e1, sa1, b1, sb1) = ops
    _lib.call("s24_spmm_pair_f8", M, N, K, F32, P(c0), P(e0), P(b0), K, P(sa0), P(sb0), P(outs[0]), N, P(rmap), 0,
              None, P(c1), P(e1), P(b1), K, P(sa1), P(sb1), P(outs[1]), M + 16, P(rmap), 1, None, 64, S())
    assert torch.equal(outs[0], refs[0]) and torch.equal(outs[1], refs[1])
    assert outs[0].abs().sum() > 0 and outs[1].abs().sum() > 0


@pytest.mark.parametrize("M,K,offset", [(128, 128, 0), (300, 512, 0), (256, 256, 2)])
def test_meta_to_f8_layout_bitwise(M, K, offset):
    """s24_meta_hw_to_f8 against the atom map restated here: f8 halfword 8 r + q
    of an atom = kind::f16 halfword at byte 2 m1 + 4 k2 + 16 m0 + 128 k1 + 256 m2
    (r = m0 + 8 m1 + 16 m2, q = k1 + 2 k2). offset != 0 runs the unaligned
    (halfword) kernel, offset 0 the 16-byte vector kernel."""
    nb = _lib.meta_hw_bytes(M, K)
    g = torch.Generator(device="cuda").manual_seed(M + K)
    src_buf = torch.randint(0, 256, (nb + offset,), dtype=torch.uint8, device="cuda", generator=g)
    dst_buf = torch.zeros(nb + offset, dtype=torch.uint8, device="cuda")
    src, dst = src_buf[offset:], dst_buf[offset:]
    _lib.call("s24_meta_hw_to_f8", P(src), M, K, P(dst), S())
    torch.cuda.synchronize()
    r = np.arange(128)[:, None]
    q = np.arange(8)[None, :]
    byte = 2 * ((r >> 3) & 1) + 4 * (q >> 1) + 16 * (r & 7) + 128 * (q & 1) + 256 * (r >> 4)
    hw = src.cpu().numpy().view(np.uint16).reshape(-1, 1024)
    want = hw[:, (byte // 2).reshape(-1)]
    got = dst.cpu().numpy().view(np.uint16).reshape(-1, 1024)
    assert np.array_equal(got, want)
