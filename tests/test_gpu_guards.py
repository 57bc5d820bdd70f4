"""Out-of-bounds write guards (compute-sanitizer is not available on the GPU
pool): the hot-path kernels write into buffers embedded in larger sentinel-
filled allocations, on ragged shapes; every byte outside the declared output
must keep its sentinel."""

import numpy as np
import pytest
import torch

from oracle import srelu24_np as O
from paper_2503_16672_b200 import _lib

from .test_gpu_kernels import BF16, F32, P, S, gpu_sparsify_token

pytestmark = pytest.mark.gpu
GUARD = 4096  # bytes of sentinel on each side


def guarded(nbytes: int, fill: int = 0xA5):
    buf = torch.full((nbytes + 2 * GUARD,), fill, dtype=torch.uint8, device="cuda")
    return buf, buf[GUARD:GUARD + nbytes]


def intact(buf, fill: int = 0xA5) -> bool:
    return bool((buf[:GUARD] == fill).all()) and bool((buf[-GUARD:] == fill).all())


def test_feature_split_x_stays_in_bounds():
    n, h = 384, 640  # 3 token blocks, 5 feature blocks
    rng = np.random.Generator(np.random.PCG64(3))
    a = O.bf16_round(np.maximum(rng.standard_normal((n, h)), 0).astype(np.float32) ** 2)
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(torch.from_numpy(a).cuda().bfloat16())
    counts = (torch.from_numpy(a).cuda() * mask.float() != 0).sum(0).cpu().numpy()
    sp, de = O.partition(counts, 0.9)
    pos = np.empty(h, np.int32)
    pos[sp] = np.arange(len(sp))
    pos[de] = -np.arange(len(de)) - 1
    rows = 2 * len(de) + len(sp)
    rp = (rows + 127) // 128 * 128
    vb, vs = guarded(rp * (n // 2) * 2)
    eb, es = guarded(_lib.meta_hw_bytes(rp, n))
    _lib.call("s24_feature_split_x", P(vals), P(meta_hw), n, h, P(torch.from_numpy(pos).cuda()), len(sp),
              len(de), P(vs), P(es), 1, None, S())
    torch.cuda.synchronize()
    assert intact(vb) and intact(eb)


def test_fp8_quantizers_stay_in_bounds():
    R, C = 100, 72
    a = torch.randn(R, C, device="cuda").bfloat16()
    cb, codes = guarded(R * C)
    sb, scales = guarded(R * 4)
    _lib.call("s24_fp8_quant_rows", P(a), BF16, R, C, C, None, 0, P(codes), C, P(scales.view(torch.float32)), None,
              0, None, 0, S())
    ld = 112
    tb, codes_t = guarded(C * ld)
    s2b, scales2 = guarded(C * 4)
    ws = torch.empty(C, dtype=torch.int32, device="cuda")
    _lib.call("s24_fp8_quant_cols_t", P(a), BF16, R, C, C, P(codes_t), ld, P(scales2.view(torch.float32)), P(ws), S())
    mb, meta8 = guarded(_lib.meta_hw_bytes(R, 256))
    src = torch.full((_lib.meta_hw_bytes(R, 256),), 0x44, dtype=torch.uint8, device="cuda")
    _lib.call("s24_meta_hw_to_f8", P(src), R, 256, P(meta8), S())
    torch.cuda.synchronize()
    assert intact(cb) and intact(sb) and intact(tb) and intact(s2b) and intact(mb)


@pytest.mark.parametrize("M", [200, 384])
def test_fwd_gemm1_and_spmm_stay_in_bounds(M):
    N, K = 512, 256  # K1: tokens M, hidden N, model K
    x = torch.randn(M, K, device="cuda").bfloat16()
    w1 = (torch.randn(K, N, device="cuda") / 16).bfloat16()
    mp = (M + 127) // 128 * 128
    vb, vals = guarded(mp * (N // 2) * 2, 0)
    eb, meta = guarded(_lib.meta_hw_bytes(M, N), 0x44)
    cnt_b, counts = guarded(N * 4, 0)
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    _lib.call("s24_fwd_gemm1_fused", P(x), K, P(w1), N, M, N, K, P(vals), P(meta), P(counts), P(stats), None, S())
    torch.cuda.synchronize()
    assert intact(vb, 0) and intact(eb, 0x44) and intact(cnt_b, 0)
    # fwd.out over the same activation, output rows through a row map, bf16
    w2 = (torch.randn(N, K, device="cuda") / 16).bfloat16()
    ob, out = guarded(M * K * 2)
    rmap = torch.randperm(M, device="cuda").int()
    _lib.call("s24_spmm", P(vals), P(meta), P(w2), 1, K, M, K, N, P(out), BF16, K, P(rmap), 0, -1, None, 0, S())
    torch.cuda.synchronize()
    assert intact(ob)
    # transposed fp32 store with paired rows (the weight-gradient epilogue)
    tb, outt = guarded(K * M * 4)
    _lib.call("s24_spmm", P(vals), P(meta), P(w2), 1, K, M, K, N, P(outt), F32, M, None, 1, -1, None, 64, S())
    torch.cuda.synchronize()
    assert intact(tb)


def test_plan_and_masked_sparsify_stay_in_bounds():
    """K7 (h not a multiple of the 1024 threads) and the masked feature-wise
    sparsifier (ragged column count) write only their declared outputs."""
    h, k = 3000, 2850
    counts = torch.randint(0, 5000, (h,), dtype=torch.int32, device="cuda")
    sb, sp = guarded(k * 4)
    db, de = guarded((h - k) * 4)
    pb, pos = guarded(h * 4)
    _lib.call("s24_plan", P(counts), h, k, P(sp), P(de), P(pos), S())
    torch.cuda.synchronize()
    assert intact(sb) and intact(db) and intact(pb)
    rows, cols = 256, 200
    a = torch.randn(rows, cols, device="cuda")
    m = (torch.rand(rows, cols, device="cuda") < 0.5).to(torch.uint8)
    cp = (cols + 127) // 128 * 128
    vb, vals = guarded(cp * (rows // 2) * 2, 0)
    mb, meta_ref = guarded((rows // 4) * cols * 2)
    hb, meta_hw = guarded(_lib.meta_hw_bytes(cols, rows), 0x44)
    kb, keep = guarded(rows * cols)
    stats = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.call("s24_sparsify_feature_masked", P(a), F32, rows, cols, cols, P(m), P(vals), P(meta_ref), P(meta_hw),
              P(keep), P(stats), S())
    torch.cuda.synchronize()
    assert intact(vb, 0) and intact(mb) and intact(hb, 0x44) and intact(kb)
