"""Interleaved A/B timing of the recipe fwd+bwd step (c2) under Python-level
switches, in one process so box-to-box and thermal drift cancel out.

usage: python scripts/ab_step.py [--blocks 8] [--steps 5] [--dense]
Variants are the `VARIANTS` dict below: name -> {module.attr: value}.
Prints median ms/step per variant (L2 flushed between steps, CUDA events).
"""

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2503_16672_b200 as s24  # noqa: E402
from paper_2503_16672_b200 import ffn as F  # noqa: E402
from paper_2503_16672_b200 import splitgemm as SG  # noqa: E402

VARIANTS = {
    "default": {},
    "unpaired": {"PAIRED_WEIGHT_GRADS": False},
    "k4_inline": {"K4_MODE": "inline"},
    "k4_inline_graph": {"K4_MODE": "inline", "_graph": True},
    "main_gathers": {"SIDE_GATHERS": False},
    "rowmap": {"ROWMAP_GEMMS": True},
    "graph": {"_graph": True},
    "act_split_bwd": {"ACT_SPLIT_IN_BWD": True},
    "k4_twice_graph": {"_k4_repeat": 2, "_graph": True},
    "fused_fw_graph": {"FUSED_FEATURE_SPLIT": True, "_graph": True},
    "nodual_graph": {"DUAL_K4": False, "_graph": True},
    "identity_graph": {"IDENTITY_LAYOUT": True, "_graph": True},
    "k4_none_graph": {"_k4_repeat": 0, "_graph": True},
    "act_split_bwd_graph": {"ACT_SPLIT_IN_BWD": True, "_graph": True},
    "act_split_bwd_k4none_graph": {"ACT_SPLIT_IN_BWD": True, "_graph": True, "_k4_repeat": 0},
    "wgrad_overlap_graph": {"WGRAD_OVERLAP": True, "_graph": True},
    "k4_gemm_graph": {"K4_MODE": "gemm", "_graph": True},
    "frame_gather_graph": {"TOKEN_ORDER_STORAGE": False, "_graph": True},
    "k4_late_graph": {"K4_AFTER_FWD_OUT": True, "_graph": True},
    "rowmap_k3_graph": {"ROWMAP_K3": True, "_graph": True},
    "rowmap_graph": {"ROWMAP_GEMMS": True, "ROWMAP_K3": True, "_graph": True},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    args = ap.parse_args()
    n, d, h = 16384, 2048, 8192
    import bench  # noqa: E402

    x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
    p = s24.FfnParams(w1=w1, w2=w2)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    names = args.variants.split(",")
    cfgs = [(nm, s24.RECIPE) for nm in names]
    if args.dense:
        cfgs.append(("dense_twin", s24.FfnConfig()))
        cfgs.append(("dense_graph", s24.FfnConfig()))
        VARIANTS["dense_graph"] = {"_graph": True}
    base = {k: getattr(F, k) for v in VARIANTS.values() for k in v if not k.startswith("_")}

    def apply(nm):
        SG.K4_REPEAT = VARIANTS.get(nm, {}).get("_k4_repeat", 1)
        for k, v in base.items():
            setattr(F, k, v)
        for k, v in VARIANTS.get(nm, {}).items():
            if not k.startswith("_"):
                setattr(F, k, v)

    graphs = {}

    def step(cfg, nm=None):
        if VARIANTS.get(nm, {}).get("_graph"):
            if nm not in graphs:
                graphs[nm] = s24.FfnStepGraph(p, cfg, n)
                graphs[nm].x.copy_(x)
                graphs[nm].dy.copy_(dy)
            graphs[nm].replay()
            return
        out, cache = s24.ffn_forward(x, p, cfg)
        s24.ffn_backward(dy, cache, p, cfg)

    for nm, cfg in cfgs:
        apply(nm)
        for _ in range(3):
            step(cfg, nm)
    torch.cuda.synchronize()
    res = {nm: [] for nm, _ in cfgs}
    clk = {nm: [] for nm, _ in cfgs}
    for _ in range(args.blocks):
        for nm, cfg in cfgs:
            apply(nm)
            sampler = bench.ClockSampler(torch.cuda.current_device())
            sampler.start()
            tot = 0.0
            evs = []
            for _ in range(args.steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                step(cfg, nm)
                e.record()
                evs.append((s, e))
            torch.cuda.synchronize()
            c = sampler.stop()
            clk[nm].append((c.get("sm_mhz") or 0, ",".join(c.get("reasons") or [])))
            tot = sum(s.elapsed_time(e) for s, e in evs)
            res[nm].append(tot / args.steps)
    print(json.dumps({nm: {"median_ms": round(statistics.median(v), 4), "min_ms": round(min(v), 4),
                           "sm_mhz": sorted(clk[nm])} for nm, v in res.items()}))


if __name__ == "__main__":
    main()
