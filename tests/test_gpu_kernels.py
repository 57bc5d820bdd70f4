"""Kernel-level parity of libs24.so on the GPU, called through the C ABI.

Bit-exact checks (masks, metadata, values given identical fp32 inputs, counts,
plans, permutation gathers) use the numpy oracle; GEMMs are checked against a
torch fp32 reference within a stated tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import srelu24_np as O
from paper_2503_16672_b200 import _lib

pytestmark = pytest.mark.gpu

F32, BF16 = 0, 1


def P(t):
    return None if t is None else t.data_ptr()


def S():
    return torch.cuda.current_stream().cuda_stream


def rel_err(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


def meta_hw_to_ref(meta_hw, rows, cols):
    ref = torch.empty(rows, cols // 4, 2, dtype=torch.uint8, device="cuda")
    _lib.call("s24_meta_hw_to_ref", P(meta_hw), rows, cols, P(ref), S())
    return ref


def gpu_sparsify_token(a, want_hw=True):
    rows, cols = a.shape
    rp = (rows + 127) // 128 * 128
    vals = torch.zeros(rp, cols // 2, dtype=torch.bfloat16, device="cuda")
    meta_ref = torch.empty(rows, cols // 4, 2, dtype=torch.uint8, device="cuda")
    meta_hw = torch.zeros(_lib.meta_hw_bytes(rows, cols), dtype=torch.uint8, device="cuda") if want_hw else None
    if meta_hw is not None:
        meta_hw.fill_(0x44)
    mask = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    dt = F32 if a.dtype == torch.float32 else BF16
    _lib.call("s24_sparsify_token", P(a), dt, rows, cols, a.stride(0), P(vals), P(meta_ref), P(meta_hw), P(mask),
              P(stats), S())
    return vals, meta_ref, meta_hw, mask, stats


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (320, 256, 448), (128, 288, 64)])
def test_dense_gemm_majors(a_mn, b_mn, M, N, K):
    torch.manual_seed(0)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    As = A.t().contiguous() if a_mn else A
    Bs = B if b_mn else B.t().contiguous()
    D = torch.empty(M, N, device="cuda")
    _lib.call("s24_gemm", P(As), a_mn, As.stride(0), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1, None,
              S())
    ref = A.float() @ B.float()
    assert rel_err(D, ref) < 1e-5


def test_dense_gemm_bf16_out_rowmap_transposed():
    torch.manual_seed(1)
    M, N, K = 200, 256, 192
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    rmap = torch.randperm(M, device="cuda").int()
    D = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    _lib.call("s24_gemm", P(A), 0, K, P(B), 1, N, M, N, K, P(D), BF16, N, P(rmap), 0, -1, None, S())
    ref = torch.empty(M, N, device="cuda")
    ref[rmap.long()] = A.float() @ B.float()
    assert rel_err(D.float(), ref) < 4e-3
    Dt = torch.zeros(N, M, device="cuda")
    _lib.call("s24_gemm", P(A), 0, K, P(B), 1, N, M, N, K, P(Dt), F32, M, P(rmap), 1, -1, None, S())
    assert rel_err(Dt.t(), ref) < 1e-5


@pytest.mark.parametrize("transposed", [0, 1])
@pytest.mark.parametrize("out_dt", [F32, BF16])
def test_gemm_splitk_rowmap(transposed, out_dt):
    """Split-K (fixed-order reduction, row map, optional transposed write) vs
    the fp32 product; the dense-remainder path of the split weight gradient."""
    torch.manual_seed(11)
    M, N, K, ks = 300, 256, 4096, 8
    A = torch.randn(M, K, device="cuda").bfloat16()   # stored MN-major, like vd
    B = torch.randn(K, N, device="cuda").bfloat16()
    rows = M + 60
    rmap = torch.randperm(rows, device="cuda")[:M].int()
    ref = torch.zeros(rows, N, device="cuda")
    ref[rmap.long()] = A.float() @ B.float()
    dt = torch.float32 if out_dt == F32 else torch.bfloat16
    D = torch.zeros((N, rows) if transposed else (rows, N), device="cuda", dtype=dt)
    ws = torch.empty(ks, M, N, device="cuda")
    _lib.call("s24_gemm_splitk", P(A), 0, K, P(B), 1, N, M, N, K, ks, P(ws), P(D), out_dt, D.shape[1], P(rmap),
              transposed, S())
    got = D.float().t() if transposed else D.float()
    assert rel_err(got, ref) < (1e-5 if out_dt == F32 else 4e-3)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_sparsify_token_matches_oracle(dtype):
    rng = np.random.Generator(np.random.PCG64(3))
    a = ((rng.random((256, 512)) < 0.3) * rng.standard_normal((256, 512))).astype(np.float32)
    a[0, :8] = [1, -2, 0, 0.5, 0, 0, 5, 0]  # KATs from ref tests/test_sparse24.py:43-57
    a[1, :4] = [1, -1, 2, 0]                 # tie KAT :59-61
    a = O.bf16_round(a)
    ta = torch.from_numpy(a).cuda().to(dtype)
    vals, meta_ref, meta_hw, mask, stats = gpu_sparsify_token(ta)
    ov, om, omask, ost = O.sparsify_token(a)
    assert np.array_equal(meta_ref.cpu().numpy(), om)
    assert np.array_equal(mask.cpu().numpy().astype(bool), omask)
    assert np.array_equal(vals[:256].float().cpu().numpy().reshape(256, 128, 2), ov)
    assert stats.cpu().tolist() == [ost["nonzeros_before"], ost["nonzeros_after"]]
    assert np.array_equal(meta_hw_to_ref(meta_hw, 256, 512).cpu().numpy(), om)


@pytest.mark.parametrize("b_mn", [1, 0])
@pytest.mark.parametrize("M,N,K", [(256, 256, 512), (384, 128, 256), (200, 384, 1024)])
def test_spmm_vs_decompressed(b_mn, M, N, K):
    torch.manual_seed(2)
    a = torch.randn(M, K, device="cuda").bfloat16()
    vals, meta_ref, meta_hw, mask, stats = gpu_sparsify_token(a)
    dense = a.float() * mask.float()
    B = torch.randn(K, N, device="cuda").bfloat16()
    Bs = B if b_mn else B.t().contiguous()
    D = torch.empty(M, N, device="cuda")
    _lib.call("s24_spmm", P(vals), P(meta_hw), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1, None, 0, S())
    ref = dense @ B.float()
    assert rel_err(D, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(256, 256, 512), (600, 384, 1024), (2600, 2048, 256), (2600, 1920, 256)])
def test_spmm_pair_matches_two_launches(M, N, K):
    """The grouped launch (two problems, one tile schedule) is bit-identical to
    two s24_spmm calls, including row maps and the transposed write. The
    larger shapes leave a partial last wave of <= 74 / 2 tiles, which runs as
    N-half units (GemmShape::tail_split) in one launch and not in the other:
    the per-element K order is the same, so the bits are too."""
    torch.manual_seed(7)
    ops = []
    for _ in range(2):
        a = torch.randn(M, K, device="cuda").bfloat16()
        vals, _, meta_hw, mask, _ = gpu_sparsify_token(a)
        ops.append((vals, meta_hw, torch.randn(K, N, device="cuda").bfloat16(), a.float() * mask.float()))
    rmap = torch.randperm(M + 40, device="cuda")[:M].int()
    ref0 = torch.zeros(M + 40, N, device="cuda")
    ref1 = torch.zeros(N, M + 40, device="cuda")
    (v0, e0, b0, a0), (v1, e1, b1, a1) = ops
    _lib.call("s24_spmm", P(v0), P(e0), P(b0), 1, N, M, N, K, P(ref0), F32, N, P(rmap), 0, -1, None, 0, S())
    _lib.call("s24_spmm", P(v1), P(e1), P(b1), 1, N, M, N, K, P(ref1), F32, M + 40, P(rmap), 1, -1, None, 0, S())
    out0, out1 = torch.zeros_like(ref0), torch.zeros_like(ref1)
    _lib.call("s24_spmm_pair", 1, M, N, K, F32, P(v0), P(e0), P(b0), N, P(out0), N, P(rmap), 0, None,
              P(v1), P(e1), P(b1), N, P(out1), M + 40, P(rmap), 1, None, 0, S())
    assert torch.equal(out0, ref0) and torch.equal(out1, ref1)
    assert rel_err(out0[rmap.long()], a0 @ b0.float()) < 1e-5
    assert rel_err(out1.t()[rmap.long()], a1 @ b1.float()) < 1e-5


def test_decompress_roundtrip():
    torch.manual_seed(4)
    a = torch.randn(128, 256, device="cuda").bfloat16()
    vals, meta_ref, meta_hw, mask, _ = gpu_sparsify_token(a)
    for mr, mh in ((meta_ref, None), (None, meta_hw)):
        out = torch.empty(128, 256, device="cuda")
        _lib.call("s24_decompress_token", P(vals), P(mr), P(mh), 128, 256, P(out), F32, 256, S())
        assert torch.equal(out, a.float() * mask.float())
    hw2 = torch.zeros_like(meta_hw)
    _lib.call("s24_meta_ref_to_hw", P(meta_ref), 128, 256, P(hw2), S())
    assert torch.equal(hw2, meta_hw)


def test_sparsify_feature_matches_oracle():
    rng = np.random.Generator(np.random.PCG64(5))
    a = O.bf16_round(((rng.random((256, 192)) < 0.3) * rng.standard_normal((256, 192))).astype(np.float32))
    ta = torch.from_numpy(a).cuda()
    rows, cols = a.shape
    vals_t = torch.zeros((cols + 127) // 128 * 128, rows // 2, dtype=torch.bfloat16, device="cuda")
    meta_ref = torch.empty(rows // 4, cols, 2, dtype=torch.uint8, device="cuda")
    meta_hw = torch.zeros(_lib.meta_hw_bytes(cols, rows), dtype=torch.uint8, device="cuda")
    mask = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.call("s24_sparsify_feature", P(ta), F32, rows, cols, cols, P(vals_t), P(meta_ref), P(meta_hw), P(mask),
              P(stats), S())
    ov, om, omask, ost = O.sparsify_feature(a)
    assert np.array_equal(meta_ref.cpu().numpy(), om)
    assert np.array_equal(mask.cpu().numpy().astype(bool), omask)
    # vals_t[j, 2g + s] == ov[g, j, s]
    assert np.array_equal(vals_t[:cols].float().cpu().numpy().reshape(cols, rows // 4, 2).transpose(1, 0, 2), ov)
    assert stats.cpu().tolist() == [ost["nonzeros_before"], ost["nonzeros_after"]]
    out = torch.empty(rows, cols, device="cuda")
    _lib.call("s24_decompress_feature", P(vals_t), None, P(meta_hw), rows, cols, P(out), F32, cols, S())
    assert np.array_equal(out.cpu().numpy(), O.decompress_feature(ov, om, rows, cols))


def test_gather_rows():
    x = torch.randn(300, 64, device="cuda").bfloat16()
    src = torch.randperm(300, device="cuda").int()
    out = torch.empty_like(x)
    _lib.call("s24_gather_rows", P(x), 300, 128, 128, P(src), P(out), 128, S())
    assert torch.equal(out, x[src.long()])


@pytest.mark.parametrize("h,ratio,hi", [(2048, 0.95, 4096), (8192, 0.95, 50), (16384, 0.95, 32768), (100, 0.5, 3),
                                        (4096, 1.0, 10), (4096, 0.0, 10), (1, 0.95, 5), (30002, 0.9, 7),
                                        (65536, 0.95, 40000), (5000, 0.95, 1 << 20)])
def test_plan_matches_oracle(h, ratio, hi):
    rng = np.random.Generator(np.random.PCG64(h))
    counts = rng.integers(0, hi, h).astype(np.int32)
    k = O.ceil_fraction(ratio, h)
    c = torch.from_numpy(counts).cuda()
    sp = torch.full((max(k, 1),), -7, dtype=torch.int32, device="cuda")
    de = torch.full((max(h - k, 1),), -7, dtype=torch.int32, device="cuda")
    pos = torch.empty(h, dtype=torch.int32, device="cuda")
    _lib.call("s24_plan", P(c), h, k, P(sp), P(de), P(pos), S())
    osp, ode = O.partition(counts, ratio)
    assert np.array_equal(sp[:k].cpu().numpy(), osp)
    assert np.array_equal(de[: h - k].cpu().numpy(), ode)
    p = pos.cpu().numpy()
    assert np.array_equal(p[osp], np.arange(k))
    assert np.array_equal(-p[ode] - 1, np.arange(h - k))


def _k1(x, w1, with_counts=True):
    M, K = x.shape
    N = w1.shape[1]
    mp = (M + 127) // 128 * 128
    vals = torch.zeros(mp, N // 2, dtype=torch.bfloat16, device="cuda")
    meta = torch.full((_lib.meta_hw_bytes(M, N),), 0x44, dtype=torch.uint8, device="cuda")
    counts = torch.zeros(N, dtype=torch.int32, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    y = torch.empty(M, N, device="cuda")
    _lib.call("s24_fwd_gemm1_fused", P(x), K, P(w1), N, M, N, K, P(vals), P(meta), P(counts) if with_counts else None,
              P(stats), P(y), S())
    return vals, meta, counts, stats, y


@pytest.mark.parametrize("M,N,K", [(256, 512, 128), (4096, 2048, 512), (200, 256, 64)])
def test_fwd_gemm1_fused_exact_given_y(M, N, K):
    x, w1, _, _ = O.synthetic_ffn_inputs(M, K, N, sparsity=0.9, seed=M)
    tx = torch.from_numpy(x).cuda().bfloat16()
    tw = torch.from_numpy(w1).cuda().bfloat16()
    vals, meta, counts, stats, y = _k1(tx, tw)
    assert rel_err(y, tx.float() @ tw.float()) < 1e-5
    yn = y.cpu().numpy()
    r = np.maximum(yn, np.float32(0))
    a = r * r
    ov, om, omask, ost = O.sparsify_token(a)
    assert np.array_equal(meta_hw_to_ref(meta, M, N).cpu().numpy(), om)
    assert np.array_equal(vals[:M].float().cpu().numpy().reshape(M, N // 4, 2), O.bf16_round(ov))
    assert np.array_equal(counts.cpu().numpy(), O.column_counts(a))
    assert stats.cpu().tolist() == [ost["nonzeros_before"], ost["nonzeros_after"], 0]


@pytest.mark.parametrize("M,N,K", [(256, 512, 128), (1024, 2048, 512)])
def test_bwd_dact_fused(M, N, K):
    x, w1, w2, dy = O.synthetic_ffn_inputs(M, K, N, sparsity=0.8, seed=7)
    tx, tw1, tw2, tg = (torch.from_numpy(t).cuda().bfloat16() for t in (x, w1, w2, dy))
    vals, meta, _, _, y = _k1(tx, tw1, with_counts=False)
    gv = torch.zeros_like(vals)
    _lib.call("s24_bwd_dact_fused", P(tg), K, P(tw2), K, M, N, K, P(vals), P(meta), P(gv), S())
    G = tg.float() @ tw2.float().t()  # [M, N]
    mref = meta_hw_to_ref(meta, M, N).long()  # [M, N/4, 2]
    Gk = torch.gather(G.view(M, N // 4, 4), 2, mref)  # [M, N/4, 2]
    av = vals[:M].float().view(M, N // 4, 2)
    expect = Gk * 2 * av.sqrt()
    assert rel_err(gv[:M].float().view(M, N // 4, 2), expect) < 5e-3


@pytest.mark.parametrize("nonneg", [0, 1])
def test_feature_split_matches_oracle(nonneg):
    """K4 against the oracle; nonneg=1 (raw-value ranking for relu^2 operands)
    on a non-negative operand with many ties must give the identical split."""
    n, h = 512, 384
    rng = np.random.Generator(np.random.PCG64(9))
    a = O.bf16_round(((rng.random((n, h)) < 0.25) * rng.standard_normal((n, h))).astype(np.float32))
    if nonneg:
        a = O.bf16_round(np.round(a * a * 4) / 4)  # >= 0, coarse values -> frequent ties
    ta = torch.from_numpy(a).cuda().bfloat16()
    vals, meta_ref, meta_hw, mask, _ = gpu_sparsify_token(ta)
    am = a * mask.cpu().numpy().astype(np.float32)
    counts = O.column_counts(am)
    ks = O.ceil_fraction(0.9, h)
    osp, ode = O.partition(counts, 0.9)
    pos = np.empty(h, np.int32)
    pos[osp] = np.arange(len(osp))
    pos[ode] = -np.arange(len(ode)) - 1
    tpos = torch.from_numpy(pos).cuda()
    sp_pad = (ks + 127) // 128 * 128
    d_pad = (h - ks + 127) // 128 * 128
    vs = torch.full((sp_pad, n // 2), 7.0, dtype=torch.bfloat16, device="cuda")
    es = torch.zeros(_lib.meta_hw_bytes(sp_pad, n), dtype=torch.uint8, device="cuda")
    vd = torch.full((d_pad, n), 7.0, dtype=torch.bfloat16, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.call("s24_feature_split", P(vals), P(meta_hw), n, h, P(tpos), ks, h - ks, P(vs), P(es), P(vd), P(stats), nonneg, -1,
              S())
    ov, om, _, ost = O.sparsify_feature(np.ascontiguousarray(am[:, osp]))
    got_meta = meta_hw_to_ref(es, sp_pad, n).cpu().numpy()  # [sp_pad, n/4, 2]
    assert np.array_equal(got_meta[:ks].transpose(1, 0, 2), om)
    got_v = vs.float().cpu().numpy().reshape(sp_pad, n // 4, 2)
    assert np.array_equal(got_v[:ks].transpose(1, 0, 2), ov)
    assert not got_v[ks:].any()
    assert np.array_equal(vd[: h - ks].float().cpu().numpy(), am[:, ode].T)
    assert not vd[h - ks:].float().any()
    assert stats.cpu().tolist() == [ost["nonzeros_before"], ost["nonzeros_after"]]


def test_feature_split_paired_layout():
    """Paired layout: dense feature r -> 2:4 rows 2r (tokens 4j, 4j+1; selector
    (0,1)) and 2r+1 (tokens 4j+2, 4j+3; selector (2,3)); sparse rank s -> row
    2*n_dense + s, identical to the separate layout's sparse rows."""
    n, h = 512, 384
    rng = np.random.Generator(np.random.PCG64(19))
    a = O.bf16_round(((rng.random((n, h)) < 0.3) * rng.standard_normal((n, h))).astype(np.float32))
    ta = torch.from_numpy(a).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    am = a * mask.cpu().numpy().astype(np.float32)
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ks, nd = len(osp), len(ode)
    pos = np.empty(h, np.int32)
    pos[osp] = np.arange(ks)
    pos[ode] = -np.arange(nd) - 1
    tpos = torch.from_numpy(pos).cuda()
    rows = 2 * nd + ks
    rp = (rows + 127) // 128 * 128
    vs = torch.full((rp, n // 2), 7.0, dtype=torch.bfloat16, device="cuda")
    es = torch.zeros(_lib.meta_hw_bytes(rp, n), dtype=torch.uint8, device="cuda")
    _lib.call("s24_feature_split", P(vals), P(meta_hw), n, h, P(tpos), ks, nd, P(vs), P(es), None, None, 0, 2 * nd,
              S())
    ov, om, _, _ = O.sparsify_feature(np.ascontiguousarray(am[:, osp]))
    got_meta = meta_hw_to_ref(es, rp, n).cpu().numpy()  # [rp, n/4, 2]
    got_v = vs.float().cpu().numpy().reshape(rp, n // 4, 2)
    assert np.array_equal(got_meta[2 * nd:rows].transpose(1, 0, 2), om)
    assert np.array_equal(got_v[2 * nd:rows].transpose(1, 0, 2), ov)
    dense = am[:, ode].T.reshape(nd, n // 4, 4)  # [nd, groups, 4 tokens]
    assert np.array_equal(got_v[0:2 * nd:2], dense[:, :, 0:2])
    assert np.array_equal(got_v[1:2 * nd:2], dense[:, :, 2:4])
    assert (got_meta[0:2 * nd:2] == np.array([0, 1])).all() and (got_meta[1:2 * nd:2] == np.array([2, 3])).all()
    assert not got_v[rows:].any()


@pytest.mark.parametrize("transposed", [0, 1])
def test_split_weight_grad_paired_layout(transposed):
    """The split weight gradient from the paired layout (one 2:4 GEMM, dense
    row pairs summed in the epilogue) matches the reference's split product
    (feature-wise 2:4 of the sparse features, dense features exact) of the
    masked operand in fp32."""
    import paper_2503_16672_b200 as s24
    from paper_2503_16672_b200.splitgemm import feature_split, split_weight_grad
    n, h, d = 1024, 512, 256
    rng = np.random.Generator(np.random.PCG64(23))
    a = O.bf16_round(((rng.random((n, h)) < 0.2) * rng.standard_normal((n, h))).astype(np.float32))
    ta = torch.from_numpy(a).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    am = a * mask.cpu().numpy().astype(np.float32)
    plan = s24.partition_features(torch.from_numpy(O.column_counts(am).astype(np.int32)).cuda(), 0.9)
    b = torch.randn(n, d, device="cuda").bfloat16()
    fs = feature_split(vals, meta_hw, n, h, plan)
    out = torch.zeros((d, h) if transposed else (h, d), device="cuda")
    split_weight_grad(fs, plan, b, n, out, transposed=bool(transposed))
    torch.cuda.synchronize()
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ref, _ = O.split_gemm_t(am, mask.cpu().numpy().astype(bool), b.float().cpu().numpy(), osp, ode, ordered=False)
    got = out.t() if transposed else out
    assert rel_err(got.cpu(), torch.from_numpy(ref)) < 1e-5


@pytest.mark.parametrize("nan", [False, True])
def test_feature_split_x_matches_reference_kernel(nan):
    """The hot-path K4x writes exactly what the reference-layout K4 writes in
    the paired layout, for the activation (>= 0, raw ranking) and for g_pre
    (magnitude keys, NaN last). With NaN among the activation's kept values,
    K1's flag switches the raw ranking back to the NaN-aware keys."""
    n, h = 512, 512
    rng = np.random.Generator(np.random.PCG64(31))
    y = O.bf16_round(rng.standard_normal((n, h)).astype(np.float32))
    act = O.bf16_round(np.maximum(y, 0) ** 2)
    if nan:
        act[rng.random((n, h)) < 0.05] = np.nan
    ta = torch.from_numpy(act).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    g = torch.randn(n, h, device="cuda").bfloat16() * mask.bfloat16()
    gvals = torch.zeros_like(vals)
    # g on the forward keep pattern, compressed with the same metadata
    _lib.call("s24_compress_token_with_mask", P(g), BF16, n, h, h, P(mask), P(gvals), None, None, None, S())
    am = np.nan_to_num(act, nan=1.0) * mask.cpu().numpy().astype(np.float32)
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ks, nd = len(osp), len(ode)
    pos = np.empty(h, np.int32)
    pos[osp] = np.arange(ks)
    pos[ode] = -np.arange(nd) - 1
    tpos = torch.from_numpy(pos).cuda()
    rows = 2 * nd + ks
    rp = (rows + 127) // 128 * 128
    flag = torch.tensor([1 if nan else 0], dtype=torch.int64, device="cuda")

    def bufs():
        return (torch.full((rp, n // 2), 7.0, dtype=torch.bfloat16, device="cuda"),
                torch.zeros(_lib.meta_hw_bytes(rp, n), dtype=torch.uint8, device="cuda"))
    for v, nn in ((vals, 1), (gvals, 0)):
        rv, re_ = bufs()
        _lib.call("s24_feature_split", P(v), P(meta_hw), n, h, P(tpos), ks, nd, P(rv), P(re_), None, None, 0,
                  2 * nd, S())
        gv_, ge = bufs()
        _lib.call("s24_feature_split_x", P(v), P(meta_hw), n, h, P(tpos), ks, nd, P(gv_), P(ge), nn, P(flag), S())
        assert torch.equal(re_, ge)
        assert torch.equal(rv.view(torch.int16), gv_.view(torch.int16))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(384, 1024), (100, 256), (4, 128)])
def test_sparsify_token_hw_fast_path_bitwise(dtype, rows, cols):
    """s24_sparsify_token with only values + hw metadata requested takes the
    sector-mapped fast kernel: bit-identical to the general kernel (which also
    writes the reference metadata and the mask), NaN / Inf and ragged row
    counts included."""
    a = torch.randn(rows, cols, device="cuda") * (torch.rand(rows, cols, device="cuda") < 0.4)
    a[torch.rand(rows, cols, device="cuda") < 0.01] = float("nan")
    a[torch.rand(rows, cols, device="cuda") < 0.005] = float("inf")
    a = a.to(dtype)
    v0, _, m0, _, s0 = gpu_sparsify_token(a)
    v1 = torch.zeros_like(v0)
    m1 = torch.full_like(m0, 0x44)
    s1 = torch.zeros(2, dtype=torch.int64, device="cuda")
    dt = F32 if dtype == torch.float32 else BF16
    _lib.call("s24_sparsify_token", P(a), dt, rows, cols, cols, P(v1), None, P(m1), None, P(s1), S())
    v2, m2 = torch.zeros_like(v0), torch.full_like(m0, 0x44)
    _lib.call("s24_sparsify_token", P(a), dt, rows, cols, cols, P(v2), None, P(m2), None, None, S())  # (no statistics)
    torch.cuda.synchronize()
    assert torch.equal(v0.view(torch.int16), v1.view(torch.int16)) and torch.equal(v0.view(torch.int16), v2.view(torch.int16))
    assert torch.equal(m0, m1) and torch.equal(m0, m2) and torch.equal(s0, s1)
