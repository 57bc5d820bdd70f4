"""Run the step's two feature-wise splits (K4 of act and g_pre) with one
build of libs24.so, for ncu captures and standalone A/B timing:
usage: python scripts/k4_probe.py [--lib path/to/libs24.so] [--iters 3]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import _lib  # noqa: E402
from paper_2503_16672_b200.splitgemm import alloc_feature_split, run_feature_split  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
if args.lib:
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from ab_step import load_lib  # noqa: E402

    _lib._lib = load_lib(args.lib)
import bench  # noqa: E402

n, d, h = 16384, 2048, 8192
x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
p = s24.FfnParams(w1=w1, w2=w2)
out, cache = s24.ffn_forward(x, p, s24.RECIPE)
grads = s24.ffn_backward(dy, cache, p, s24.RECIPE)
plan, npad = cache.plan, cache.act_vals.shape[0]
g_vals = grads.g_pre_sparse.data
fa = alloc_feature_split(cache.act_vals, cache.act_meta, npad, h, plan)
fg = alloc_feature_split(g_vals, cache.act_meta, npad, h, plan)
torch.cuda.synchronize()
for _ in range(args.iters):
    run_feature_split(fa, cache.act_vals, cache.act_meta, npad, h, plan, nonneg=True, nan_flag=cache.stats_dev[2:])
    run_feature_split(fg, g_vals, cache.act_meta, npad, h, plan)
torch.cuda.synchronize()
print("ok")
