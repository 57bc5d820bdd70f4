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


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(512, 1024, 256), (320, 800, 448), (128, 288, 64)])
def test_wide_dense_tiles_bitwise_equal_narrow(monkeypatch, a_mn, b_mn, M, N, K):
    """256x512 tiles (two N=256 MMAs per k-step, one 512-column accumulator)
    vs 256x256: same per-element K order, so the results are bit-identical;
    also K1's fused epilogue (metadata gathered per atom) under both."""
    torch.manual_seed(3)
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    As = A.t().contiguous() if a_mn else A
    Bs = B if b_mn else B.t().contiguous()
    outs = []
    for bn in ("256", "512"):
        monkeypatch.setenv("S24_DENSE_BN", bn)
        D = torch.full((M, N), float("nan"), device="cuda")
        _lib.call("s24_gemm", P(As), a_mn, As.stride(0), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0,
                  -1, None, S())
        outs.append(D)
    assert torch.equal(outs[0], outs[1])
    assert rel_err(outs[1], A.float() @ B.float()) < 1e-5
    if not a_mn and b_mn and N % 128 == 0:
        res = []
        for bn in ("256", "512"):
            monkeypatch.setenv("S24_DENSE_BN", bn)
            vals = torch.zeros((M + 127) // 128 * 128, N // 2, device="cuda", dtype=torch.bfloat16)
            meta = torch.full((_lib.meta_hw_bytes(M, N),), 0x44, device="cuda", dtype=torch.uint8)
            counts = torch.zeros(N, device="cuda", dtype=torch.int32)
            stats = torch.zeros(2, device="cuda", dtype=torch.int64)
            _lib.call("s24_fwd_gemm1_fused", P(A), K, P(B), N, M, N, K, P(vals), P(meta), P(counts), P(stats), None,
                      None, None, None, 0, None, S())
            res.append((vals, meta, counts, stats))
        for x, y in zip(*res):
            assert torch.equal(x, y)


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
@pytest.mark.parametrize("tail", ["1", "0"])
def test_spmm_pair_matches_two_launches(monkeypatch, M, N, K, tail):
    """The grouped launch (two problems, one tile schedule) is bit-identical to
    two s24_spmm calls, including row maps and the transposed write. The
    larger shapes leave a partial last wave of <= 74 / 2 tiles, which runs as
    N-half units (GemmShape::tail_split) unless S24_TAIL_SPLIT=0; the
    references always run without it."""
    torch.manual_seed(7)
    monkeypatch.setenv("S24_TAIL_SPLIT", "0")
    ops = []
    for _ in range(2):
        a = torch.randn(M, K, device="cuda").bfloat16()
        vals, _, meta_hw, _, _ = gpu_sparsify_token(a)
        ops.append((vals, meta_hw, torch.randn(K, N, device="cuda").bfloat16()))
    rmap = torch.randperm(M + 40, device="cuda")[:M].int()
    ref0 = torch.zeros(M + 40, N, device="cuda")
    ref1 = torch.zeros(N, M + 40, device="cuda")
    (v0, e0, b0), (v1, e1, b1) = ops
    _lib.call("s24_spmm", P(v0), P(e0), P(b0), 1, N, M, N, K, P(ref0), F32, N, P(rmap), 0, -1, None, 0, S())
    _lib.call("s24_spmm", P(v1), P(e1), P(b1), 1, N, M, N, K, P(ref1), F32, M + 40, P(rmap), 1, -1, None, 0, S())
    torch.cuda.synchronize()
    monkeypatch.setenv("S24_TAIL_SPLIT", tail)
    out0, out1 = torch.zeros_like(ref0), torch.zeros_like(ref1)
    _lib.call("s24_spmm_pair", 1, M, N, K, F32, P(v0), P(e0), P(b0), N, P(out0), N, P(rmap), 0, None,
              P(v1), P(e1), P(b1), N, P(out1), M + 40, P(rmap), 1, None, 0, S())
    assert torch.equal(out0, ref0) and torch.equal(out1, ref1)
    assert out0.abs().sum() > 0 and out1.abs().sum() > 0
    # single launches with the tail split (bf16 out, no row map) vs without
    outs = []
    for tl in ("0", tail):
        monkeypatch.setenv("S24_TAIL_SPLIT", tl)
        o = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        _lib.call("s24_spmm", P(v0), P(e0), P(b0), 1, N, M, N, K, P(o), BF16, N, None, 0, -1, None, 0, S())
        outs.append(o)
    assert torch.equal(outs[0], outs[1])


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
                                        (4096, 1.0, 10), (4096, 0.0, 10), (1, 0.95, 5)])
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


def _k1(x, w1, with_counts=True, row_map=None):
    M, K = x.shape
    N = w1.shape[1]
    mp = (M + 127) // 128 * 128
    vals = torch.zeros(mp, N // 2, dtype=torch.bfloat16, device="cuda")
    meta = torch.full((_lib.meta_hw_bytes(M, N),), 0x44, dtype=torch.uint8, device="cuda")
    counts = torch.zeros(N, dtype=torch.int32, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    y = torch.empty(M, N, device="cuda")
    _lib.call("s24_fwd_gemm1_fused", P(x), K, P(w1), N, M, N, K, P(vals), P(meta), P(counts) if with_counts else None,
              P(stats), P(y), None, None, None, 0, P(row_map), S())
    return vals, meta, counts, stats, y


@pytest.mark.parametrize("M", [512, 300])
def test_k1_k3_row_map_equals_gathered_input(M):
    """The token permutation applied in the K1 / K3 epilogues (row map) is
    bit-identical to gathering the rows first (ref matcore.py:291-296)."""
    N, K = 512, 256
    x, w1, w2, dy = O.synthetic_ffn_inputs(M, K, N, sparsity=0.85, seed=3)
    tx, tw1, tw2, tg = (torch.from_numpy(t).cuda().bfloat16() for t in (x, w1, w2, dy))
    perm = torch.from_numpy(O.make_permutation(5, M).astype(np.int32)).cuda()
    inv = torch.empty_like(perm)
    inv[perm.long()] = torch.arange(M, dtype=torch.int32, device="cuda")
    xg, gg = tx[inv.long()], tg[inv.long()]  # x_in[perm[r]] = x[r]
    v0, m0, c0, s0, y0 = _k1(xg, tw1)
    v1, m1, c1, s1, y1 = _k1(tx, tw1, row_map=perm)
    assert torch.equal(v0, v1) and torch.equal(m0, m1) and torch.equal(c0, c1) and torch.equal(s0, s1)
    assert torch.equal(y0, y1)
    g0, g1 = torch.zeros_like(v0), torch.zeros_like(v0)
    _lib.call("s24_bwd_dact_fused", P(gg), K, P(tw2), K, M, N, K, P(v0), P(m0), P(g0), None, None, None, 0, None, S())
    _lib.call("s24_bwd_dact_fused", P(tg), K, P(tw2), K, M, N, K, P(v0), P(m0), P(g1), None, None, None, 0, P(perm),
              S())
    assert torch.equal(g0, g1) and g0.abs().sum() > 0


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
    assert stats.cpu().tolist() == [ost["nonzeros_before"], ost["nonzeros_after"]]


@pytest.mark.parametrize("M,N,K", [(256, 512, 128), (1024, 2048, 512)])
def test_bwd_dact_fused(M, N, K):
    x, w1, w2, dy = O.synthetic_ffn_inputs(M, K, N, sparsity=0.8, seed=7)
    tx, tw1, tw2, tg = (torch.from_numpy(t).cuda().bfloat16() for t in (x, w1, w2, dy))
    vals, meta, _, _, y = _k1(tx, tw1, with_counts=False)
    gv = torch.zeros_like(vals)
    _lib.call("s24_bwd_dact_fused", P(tg), K, P(tw2), K, M, N, K, P(vals), P(meta), P(gv), None, None, None, 0, None, S())
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


@pytest.mark.parametrize("layout", ["paired", "identity"])
@pytest.mark.parametrize("transposed", [0, 1])
def test_split_weight_grad_paired_equals_separate(transposed, layout):
    """The split weight gradient from the paired layout (one 2:4 GEMM, row
    pairs summed in the epilogue) matches the separate sparse + dense GEMMs
    and the fp32 product of the masked operand."""
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
    outs = []
    for paired in (False, True):
        fs = feature_split(vals, meta_hw, n, h, plan, paired=paired, identity=paired and layout == "identity")
        out = torch.zeros((d, h) if transposed else (h, d), device="cuda")
        split_weight_grad(fs, plan, b, n, out, transposed=bool(transposed))
        outs.append(out.t() if transposed else out)
    torch.cuda.synchronize()
    # reference: feature-wise 2:4 of the sparse features, dense features exact
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ref, _ = O.split_gemm_t(am, mask.cpu().numpy().astype(bool), b.float().cpu().numpy(), osp, ode, ordered=False)
    for o in outs:
        assert rel_err(o.cpu(), torch.from_numpy(ref)) < 1e-5
    assert rel_err(outs[1], outs[0]) < 1e-6


@pytest.mark.parametrize("nonneg", [0, 1])
def test_feature_split_identity_layout(nonneg):
    """Identity layout (coalesced K4): dense pairs, zero padding to 128 rows,
    then feature f at row pad + f with the oracle's feature-wise 2:4."""
    n, h = 512, 384
    rng = np.random.Generator(np.random.PCG64(29))
    a = O.bf16_round(((rng.random((n, h)) < 0.3) * rng.standard_normal((n, h))).astype(np.float32))
    if nonneg:
        a = O.bf16_round(np.round(a * a * 4) / 4)
    ta = torch.from_numpy(a).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    am = a * mask.cpu().numpy().astype(np.float32)
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ks, nd = len(osp), len(ode)
    pos = np.empty(h, np.int32)
    pos[osp] = np.arange(ks)
    pos[ode] = -np.arange(nd) - 1
    pad = (2 * nd + 127) // 128 * 128
    rows = pad + h
    vs = torch.full((rows, n // 2), 7.0, dtype=torch.bfloat16, device="cuda")
    es = torch.zeros(_lib.meta_hw_bytes(rows, n), dtype=torch.uint8, device="cuda")
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.call("s24_feature_split_id", P(vals), P(meta_hw), n, h, P(torch.from_numpy(pos).cuda()), nd, P(vs), P(es),
              P(stats), nonneg, S())
    ov, om, _, ost = O.sparsify_feature(am)  # every feature
    got_meta = meta_hw_to_ref(es, rows, n).cpu().numpy()
    got_v = vs.float().cpu().numpy().reshape(rows, n // 4, 2)
    assert np.array_equal(got_meta[pad:].transpose(1, 0, 2), om)
    assert np.array_equal(got_v[pad:].transpose(1, 0, 2), ov)
    dense = am[:, ode].T.reshape(nd, n // 4, 4)
    assert np.array_equal(got_v[0:2 * nd:2], dense[:, :, 0:2])
    assert np.array_equal(got_v[1:2 * nd:2], dense[:, :, 2:4])
    assert (got_meta[0:2 * nd:2] == np.array([0, 1])).all() and (got_meta[1:2 * nd:2] == np.array([2, 3])).all()
    assert not got_v[2 * nd:pad].any()
    _, _, _, ost_s = O.sparsify_feature(np.ascontiguousarray(am[:, osp]))
    assert stats.cpu().tolist() == [ost_s["nonzeros_before"], ost_s["nonzeros_after"]]


@pytest.mark.parametrize("dual", [False, True])
def test_feature_split_x_matches_reference_kernel(dual):
    """The hot-path K4x (one or two operands sharing the keep pattern) writes
    exactly what the reference-layout K4 writes in the paired layout."""
    n, h = 512, 512
    rng = np.random.Generator(np.random.PCG64(31))
    y = O.bf16_round(rng.standard_normal((n, h)).astype(np.float32))
    act = O.bf16_round(np.maximum(y, 0) ** 2)
    ta = torch.from_numpy(act).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    g = torch.randn(n, h, device="cuda").bfloat16() * mask.bfloat16()
    gvals = torch.zeros_like(vals)
    # g on the forward keep pattern, compressed with the same metadata
    _lib.call("s24_compress_token_with_mask", P(g), BF16, n, h, h, P(mask), P(gvals), None, None, None, S())
    am = act * mask.cpu().numpy().astype(np.float32)
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ks, nd = len(osp), len(ode)
    pos = np.empty(h, np.int32)
    pos[osp] = np.arange(ks)
    pos[ode] = -np.arange(nd) - 1
    tpos = torch.from_numpy(pos).cuda()
    rows = 2 * nd + ks
    rp = (rows + 127) // 128 * 128

    def bufs():
        return (torch.full((rp, n // 2), 7.0, dtype=torch.bfloat16, device="cuda"),
                torch.zeros(_lib.meta_hw_bytes(rp, n), dtype=torch.uint8, device="cuda"))
    ref = []
    for v, nn in ((vals, 1), (gvals, 0)):
        vs, es = bufs()
        _lib.call("s24_feature_split", P(v), P(meta_hw), n, h, P(tpos), ks, nd, P(vs), P(es), None, None, nn,
                  2 * nd, S())
        ref.append((vs, es))
    va, ea = bufs()
    vb, eb = bufs()
    if dual:
        _lib.call("s24_feature_split_x", P(vals), P(gvals), P(meta_hw), n, h, P(tpos), ks, nd, P(va), P(ea), P(vb),
                  P(eb), 1, None, S())
        got = [(va, ea), (vb, eb)]
    else:
        _lib.call("s24_feature_split_x", P(vals), None, P(meta_hw), n, h, P(tpos), ks, nd, P(va), P(ea), None, None,
                  1, None, S())
        _lib.call("s24_feature_split_x", P(gvals), None, P(meta_hw), n, h, P(tpos), ks, nd, P(vb), P(eb), None, None,
                  0, None, S())
        got = [(va, ea), (vb, eb)]
    for (rv, re_), (gv_, ge) in zip(ref, got):
        assert torch.equal(rv, gv_) and torch.equal(re_, ge)


@pytest.mark.parametrize("M,N,K,b_mn", [(1024, 2048, 1024, 1), (640, 256, 512, 1), (768, 4096, 512, 0),
                                        (512, 512, 1024, 0)])
def test_spmm_fs_equals_spmm_plus_feature_split(M, N, K, b_mn):
    """s24_spmm_fs (the 2:4 GEMM whose CTAs also split their own A stages
    feature-wise) = s24_spmm + s24_feature_split_x, bit for bit; both operand
    kinds (act >= 0 ranked raw, g_pre ranked by |x| with NaN keys)."""
    rng = np.random.Generator(np.random.PCG64(M + N))
    npad = (M + 127) // 128 * 128
    for nonneg in (1, 0):
        y = O.bf16_round(rng.standard_normal((M, K)).astype(np.float32))
        a_np = O.bf16_round(np.maximum(y, 0) ** 2) if nonneg else y
        ta = torch.from_numpy(a_np).cuda().bfloat16()
        vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
        am = np.abs(a_np) * mask.cpu().numpy().astype(np.float32)
        osp, ode = O.partition(O.column_counts(am), 0.9)
        ks, nd = len(osp), len(ode)
        pos = np.empty(K, np.int32)
        pos[osp] = np.arange(ks)
        pos[ode] = -np.arange(nd) - 1
        tpos = torch.from_numpy(pos).cuda()
        rp = (2 * nd + ks + 127) // 128 * 128
        B = torch.randn(K, N, device="cuda").bfloat16()
        Bs = B if b_mn else B.t().contiguous()
        vp = torch.zeros(npad, K // 2, dtype=torch.bfloat16, device="cuda")
        vp[:M] = vals[:M]
        mp = torch.full((_lib.meta_hw_bytes(npad, K),), 0x44, dtype=torch.uint8, device="cuda")
        mp[:meta_hw.numel()] = meta_hw
        outs = []
        for fused in (False, True):
            vs = torch.full((rp, npad // 2), 7.0, dtype=torch.bfloat16, device="cuda")
            es = torch.zeros(_lib.meta_hw_bytes(rp, npad), dtype=torch.uint8, device="cuda")
            D = torch.zeros(M, N, device="cuda")
            if fused:
                _lib.call("s24_spmm_fs", P(vp), P(mp), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1,
                          None, npad, P(tpos), ks, nd, P(vs), P(es), nonneg, S())
            else:
                _lib.call("s24_spmm", P(vp), P(mp), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1,
                          None, 0, S())
                _lib.call("s24_feature_split_x", P(vp), None, P(mp), npad, K, P(tpos), ks, nd, P(vs), P(es), None,
                          None, nonneg, None, S())
            torch.cuda.synchronize()
            outs.append((D, vs, es))
        (d0, v0, e0), (d1, v1, e1) = outs
        assert torch.equal(d0, d1)
        if not torch.equal(v0, v1):
            bad = (v0 != v1).nonzero()
            print("mismatch", nonneg, bad.shape[0], bad[:6].tolist(), v0[bad[:6, 0], bad[:6, 1]].tolist(),
                  v1[bad[:6, 0], bad[:6, 1]].tolist(), "rows", torch.unique(bad[:, 0]).tolist()[:10], 2 * nd, ks)
        assert torch.equal(v0, v1), ("vs", nonneg)
        assert torch.equal(e0, e1), ("es", nonneg)
