"""Run one c2-shaped GEMM of the step repeatedly (for ncu captures):
usage: python scripts/gemm_probe.py {k1|k1nc|k3|relu2|dact|fwdout|dx|dw|dense|k4|gather|plan}[,...] [--iters 5]
--time prints the median CUDA-event time per call instead; with S24_LIB pointing at an
S24_PROBE build (MMA-only / feed-only, csrc/gemm.cuh) it gives profiles/r02/gemm_ceilings_c2.txt.
ncu: the step that builds the operands launches 6 gemm_kernel, 2 k_feature_split_x, 2 k_gather_rows and
1 k_plan first (skip them with -s)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("which")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--time", action="store_true", help="print the median CUDA-event time per call")
args = ap.parse_args()
import bench  # noqa: E402

n, d, h = 16384, 2048, 8192
x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
p = s24.FfnParams(w1=w1, w2=w2)
out, cache = s24.ffn_forward(x, p, s24.RECIPE)
g = s24.ffn_backward(dy, cache, p, s24.RECIPE)
torch.cuda.synchronize()
S = torch.cuda.current_stream().cuda_stream
P = lambda t: t.data_ptr()  # noqa: E731
o = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
dw = torch.empty(h, d, device="cuda")
gv = torch.empty_like(cache.act_vals)
if args.which in ("relu2", "dact"):  # dense twin operands: act / g_pre [n, h]
    gv = torch.randn(n, h, device="cuda").bfloat16().relu_()
    gv2 = torch.empty_like(gv)
stats = torch.zeros(3, dtype=torch.int64, device="cuda")
cnt = torch.zeros(h, dtype=torch.int32, device="cuda")
av = torch.empty_like(cache.act_vals)
am = torch.empty_like(cache.act_meta)
fa, plan = cache.act_split, cache.plan
calls = {
    "k1": lambda: _lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(av), P(am), P(cnt), P(stats), None, S),
    "k1nc": lambda: _lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(av), P(am), None, None, None, S),
    "k3": lambda: _lib.call("s24_bwd_dact_fused", P(dy), d, P(w2), d, n, h, d, P(cache.act_vals), P(cache.act_meta),
                            P(gv), S),
    "fwdout": lambda: _lib.call("s24_spmm", P(cache.act_vals), P(cache.act_meta), P(w2), 1, d, n, d, h, P(o), 1, d,
                                None, 0, -1, None, 0, S),
    "dx": lambda: _lib.call("s24_spmm", P(cache.act_vals), P(cache.act_meta), P(w1), 0, h, n, d, h, P(o), 1, d,
                            None, 0, -1, None, 0, S),
    "dw": lambda: _lib.call("s24_spmm", P(fa.vs), P(fa.es), P(dy), 1, d, fa.rows(plan), d, n, P(dw), 0, d,
                            P(plan.paired_row_map), 0, fa.rows(plan), None, fa.pair_rows, S),
    "relu2": lambda: _lib.call("s24_gemm_relu2", P(x), d, P(w1), h, n, h, d, P(gv), h, S),
    "dact": lambda: _lib.call("s24_gemm_dact", P(dy), d, P(w2), d, n, h, d, P(gv), h, P(gv2), h, S),
    "dense": lambda: _lib.call("s24_gemm", P(x), 0, d, P(w1), 1, h, n, h, d, P(gv), 1, h, None, 0, -1, None, S),
    "k4": lambda: _lib.call("s24_feature_split_x", P(cache.act_vals), P(cache.act_meta), n, h, P(plan.feat_pos),
                            plan.n_sparse, plan.n_dense, P(fa.vs), P(fa.es), 1, None, S),
    "gather": lambda: _lib.call("s24_gather_rows", P(x), n, 2 * d, 2 * d, P(cache.inv_dev), P(o), 2 * d, S),
    "plan": lambda: _lib.call("s24_plan", P(cache.counts), h, plan.n_sparse, P(plan.sparse_features),
                              P(plan.dense_features), P(plan.feat_pos), S),
}
for which in args.which.split(","):
    if args.time:
        ts = []
        for _ in range(args.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            calls[which]()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"{which} median_ms {ts[len(ts) // 2]:.4f} min_ms {ts[0]:.4f}")
        continue
    for _ in range(args.iters):
        calls[which]()
torch.cuda.synchronize()
print("ok", args.which)
