"""Recipe step in bf16 vs the e4m3 configurations (fp8_emulation, +
fp8_backward) at one bench shape: CUDA-graph replays, L2 flushed between
steps, interleaved rounds; then a traced eager pass of the fp8 step for the
per-kernel breakdown.

usage: python scripts/fp8_step.py [--config c2] [--steps 5] [--rounds 3]
"""

import argparse
import json
import statistics
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    n, d, h = bench.CONFIGS[args.config]
    x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
    p = s24.FfnParams(w1=w1, w2=w2)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    cfgs = {
        "bf16_recipe": s24.RECIPE,
        "fp8_fwd_recipe": replace(s24.RECIPE, fp8_emulation=True),
        "fp8_all_recipe": replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True),
        "bf16_dense": s24.FfnConfig(),
        "fp8_all_dense": s24.FfnConfig(fp8_emulation=True, fp8_backward=True),
    }
    graphs = {}
    for k, cfg in cfgs.items():
        g = s24.FfnStepGraph(p, cfg, n)
        g.x.copy_(x)
        g.dy.copy_(dy)
        graphs[k] = g
    times = {k: [] for k in cfgs}
    for _ in range(args.rounds):
        for k, g in graphs.items():
            for _ in range(2):
                g.replay()
            tot = 0.0
            for _ in range(args.steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                g.replay()
                e.record()
                e.synchronize()
                tot += s.elapsed_time(e)
            times[k].append(tot / args.steps)
    res = {k: statistics.median(v) for k, v in times.items()}
    res["speedup_fp8_all_vs_bf16_recipe"] = res["bf16_recipe"] / res["fp8_all_recipe"]
    res["speedup_fp8_all_recipe_vs_bf16_dense"] = res["bf16_dense"] / res["fp8_all_recipe"]
    res["speedup_fp8_recipe_vs_fp8_dense"] = res["fp8_all_dense"] / res["fp8_all_recipe"]
    print(json.dumps({"config": args.config, "ms_per_step": res}), flush=True)
    # per-kernel breakdown of the fp8 recipe step (eager, traced)
    for name in ("fp8_all_recipe",):
        cfg = cfgs[name]
        tr = bench.KernelTracer(torch)
        for _ in range(2):
            out, cache = s24.ffn_forward(x, p, cfg)
            s24.ffn_backward(dy, cache, p, cfg)
        torch.cuda.synchronize()
        _lib.set_tracer(tr)
        for _ in range(args.steps):
            flush.zero_()
            out, cache = s24.ffn_forward(x, p, cfg)
            s24.ffn_backward(dy, cache, p, cfg)
        _lib.set_tracer(None)
        torch.cuda.synchronize()
        agg = tr.summary()
        print(f"\n{name}: per-kernel (eager, traced), ms/step")
        for label, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
            ms = a["ms"] / args.steps
            if a["kind"] in ("tensor_f8", "tensor_f8_sparse", "tensor", "tensor_sparse"):
                rate = f"{a['work'] / (a['ms'] / 1e3) / 1e12:8.0f} TF/s"
            elif a["kind"] == "hbm":
                rate = f"{a['work'] / (a['ms'] / 1e3) / 1e9:8.0f} GB/s"
            else:
                rate = ""
            print(f"  {ms:7.3f}  x{a['launches'] // args.steps:<2} {rate:>14}  {label}")


if __name__ == "__main__":
    main()
