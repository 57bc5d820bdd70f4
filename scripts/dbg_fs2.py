import sys
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import srelu24_np as O
from paper_2503_16672_b200 import _lib
from tests.test_gpu_kernels import P, S, F32, gpu_sparsify_token
fails = 0
for trial in range(24):
    M, N, K, b_mn = [(1024, 2048, 1024, 1), (640, 256, 512, 1), (768, 4096, 512, 0), (512, 512, 1024, 0)][trial % 4]
    rng = np.random.Generator(np.random.PCG64(1000 + trial))
    npad = (M + 127) // 128 * 128
    nonneg = trial % 2
    y = O.bf16_round(rng.standard_normal((M, K)).astype(np.float32))
    a_np = O.bf16_round(np.maximum(y, 0) ** 2) if nonneg else y
    ta = torch.from_numpy(a_np).cuda().bfloat16()
    vals, _, meta_hw, mask, _ = gpu_sparsify_token(ta)
    am = np.abs(a_np) * mask.cpu().numpy().astype(np.float32)
    osp, ode = O.partition(O.column_counts(am), 0.9)
    ks, nd = len(osp), len(ode)
    pos = np.empty(K, np.int32); pos[osp] = np.arange(ks); pos[ode] = -np.arange(nd) - 1
    tpos = torch.from_numpy(pos).cuda()
    rp = (2 * nd + ks + 127) // 128 * 128
    B = torch.randn(K, N, device="cuda").bfloat16()
    Bs = B if b_mn else B.t().contiguous()
    vp = torch.zeros(npad, K // 2, dtype=torch.bfloat16, device="cuda"); vp[:M] = vals[:M]
    mp = torch.full((_lib.meta_hw_bytes(npad, K),), 0x44, dtype=torch.uint8, device="cuda"); mp[:meta_hw.numel()] = meta_hw
    outs = []
    for fused in (False, True, True, True):
        vs = torch.full((rp, npad // 2), 7.0, dtype=torch.bfloat16, device="cuda")
        es = torch.zeros(_lib.meta_hw_bytes(rp, npad), dtype=torch.uint8, device="cuda")
        D = torch.zeros(M, N, device="cuda")
        if fused:
            _lib.call("s24_spmm_fs", P(vp), P(mp), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1, None, npad, P(tpos), ks, nd, P(vs), P(es), nonneg, S())
        else:
            _lib.call("s24_spmm", P(vp), P(mp), P(Bs), b_mn, Bs.stride(0), M, N, K, P(D), F32, N, None, 0, -1, None, 0, S())
            _lib.call("s24_feature_split_x", P(vp), None, P(mp), npad, K, P(tpos), ks, nd, P(vs), P(es), None, None, nonneg, S())
        torch.cuda.synchronize()
        outs.append((D, vs, es))
    d0, v0, e0 = outs[0]
    for i, (d1, v1, e1) in enumerate(outs[1:]):
        ok = torch.equal(d0, d1), torch.equal(v0, v1), torch.equal(e0, e1)
        if not all(ok):
            fails += 1
            bad = (v0 != v1).nonzero()
            print("trial", trial, (M, N, K, b_mn, nonneg), "rep", i, ok, bad.shape[0], bad[:4].tolist(),
                  "rows", torch.unique(bad[:, 0]).tolist()[:8], "tokcols", torch.unique(bad[:, 1] // 64).tolist()[:8], 2 * nd, ks)
print("fails", fails)
