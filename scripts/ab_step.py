"""Interleaved A/B timing of the recipe fwd+bwd step (c2 by default) across
builds of libs24.so, in one process so box-to-box and clock drift cancel out.

usage: python scripts/ab_step.py --libs paper_2503_16672_b200/libs24.so,/tmp/alt.so [--blocks 8] [--steps 5]
       [--dense] [--k4] [--n 16384 --d 2048 --h 8192]
A variant may carry environment settings read by the Python layer while the
graph is captured: --libs "a.so,a.so|S24_FOO=1".

Each library is loaded side by side (ctypes) and the whole step is captured
as a CUDA graph per library (FfnStepGraph), so a graph replays exactly that
build's kernels. Build alternatives with
`python -m paper_2503_16672_b200.build -D NAME=VALUE --out /tmp/alt.so`.
Prints median / min ms per variant (L2 flushed between steps, CUDA events)
with the SM clocks seen during each variant's blocks.
"""

import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import _lib  # noqa: E402


def load_lib(path: str) -> ctypes.CDLL:
    lib = ctypes.CDLL(str(Path(path).resolve()))
    for name, argtypes in _lib.SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _lib._RESTYPES.get(name, _lib.INT)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default=str(_lib.LIB_PATH))
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--dense", action="store_true", help="also time the dense twin (first library)")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--h", type=int, default=8192)
    ap.add_argument("--k4", action="store_true",
                    help="time only the two feature-wise splits (K4 of act and g_pre, alone) per library")
    ap.add_argument("--sparsify", action="store_true",
                    help="time only the standalone token-wise sparsifier on an [n, h] bf16 activation per library")
    args = ap.parse_args()
    import bench  # noqa: E402

    n, d, h = args.n, args.d, args.h
    x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
    p = s24.FfnParams(w1=w1, w2=w2)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    variants = []
    import os

    envs = []
    for i, spec in enumerate(args.libs.split(",")):
        path, *kv = spec.split("|")
        variants.append((f"{i}:{Path(path).name}" + ("|" + "|".join(kv) if kv else ""), load_lib(path), s24.RECIPE))
        envs.append(dict(e.split("=", 1) for e in kv))
    if args.dense:
        variants.append(("dense_twin", variants[0][1], s24.FfnConfig()))
        envs.append({})
    graphs = []
    if args.k4:
        from paper_2503_16672_b200.splitgemm import alloc_feature_split, run_feature_split

        _lib._lib = variants[0][1]
        out, cache = s24.ffn_forward(x, p, s24.RECIPE)
        grads = s24.ffn_backward(dy, cache, p, s24.RECIPE)
        plan, npad = cache.plan, cache.act_vals.shape[0]
        g_vals = grads.g_pre_sparse.data
        torch.cuda.synchronize()
    if args.sparsify:
        act = (torch.randn(n, args.h, device="cuda") * (torch.rand(n, args.h, device="cuda") < 0.1)).bfloat16()
        sv = torch.zeros(n, args.h // 2, dtype=torch.bfloat16, device="cuda")
        sm = torch.empty(_lib.meta_hw_bytes(n, args.h), dtype=torch.uint8, device="cuda")
    for (name, lib, cfg), env in zip(variants, envs):
        _lib._lib = lib
        if args.sparsify:
            g = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                _lib.call("s24_sparsify_token", act.data_ptr(), _lib.BF16, n, args.h, args.h, sv.data_ptr(), None,
                          sm.data_ptr(), None, None, st.cuda_stream)
            torch.cuda.current_stream().wait_stream(st)
            with torch.cuda.graph(g):
                _lib.call("s24_sparsify_token", act.data_ptr(), _lib.BF16, n, args.h, args.h, sv.data_ptr(), None,
                          sm.data_ptr(), None, None, torch.cuda.current_stream().cuda_stream)
            graphs.append(g)
            continue
        if args.k4:
            fa = alloc_feature_split(cache.act_vals, cache.act_meta, npad, args.h, plan)
            fg = alloc_feature_split(g_vals, cache.act_meta, npad, args.h, plan)
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                run_feature_split(fa, cache.act_vals, cache.act_meta, npad, args.h, plan, nonneg=True,
                                  nan_flag=cache.stats_dev[2:])
                run_feature_split(fg, g_vals, cache.act_meta, npad, args.h, plan)
            torch.cuda.current_stream().wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run_feature_split(fa, cache.act_vals, cache.act_meta, npad, args.h, plan, nonneg=True,
                                  nan_flag=cache.stats_dev[2:])
                run_feature_split(fg, g_vals, cache.act_meta, npad, args.h, plan)
            graphs.append(g)
            continue
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        g = s24.FfnStepGraph(p, cfg, n)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        g.x.copy_(x)
        g.dy.copy_(dy)
        graphs.append(g)
    torch.cuda.synchronize()
    res = {v[0]: [] for v in variants}
    clk = {v[0]: [] for v in variants}
    for _ in range(args.blocks):
        for (name, _, _), g in zip(variants, graphs):
            sampler = bench.ClockSampler(torch.cuda.current_device())
            sampler.start()
            evs = []
            for _ in range(args.steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                g.replay()
                e.record()
                evs.append((s, e))
            torch.cuda.synchronize()
            c = sampler.stop()
            clk[name].append(c.get("sm_mhz") or 0)
            res[name].append(sum(s.elapsed_time(e) for s, e in evs) / args.steps)
    print(json.dumps({nm: {"median_ms": round(statistics.median(v), 4), "min_ms": round(min(v), 4),
                           "sm_mhz": sorted(clk[nm])} for nm, v in res.items()}))


if __name__ == "__main__":
    main()
