"""The dense FFN step's six GEMMs (c2 shapes by default) on cuBLAS (torch.matmul,
bf16 operands, fp32 accumulation, bf16 out) against this repo's dense twin
step, both as CUDA graphs, blocks interleaved: a check that the bench's dense
denominator is not built on a weak GEMM. The cuBLAS number is GEMMs only (no
relu^2 / derivative passes, which the twin fuses), so it is a lower bound on
any dense step made of cuBLAS calls.

usage: python scripts/cublas_twin.py [--n 16384 --d 2048 --h 8192] [--steps 20] [--blocks 6]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2503_16672_b200 as s24  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--h", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--blocks", type=int, default=6)
    args = ap.parse_args()
    import bench  # noqa: E402

    n, d, h = args.n, args.d, args.h
    x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
    act = torch.randn(n, h, device="cuda").bfloat16()
    g = torch.randn(n, h, device="cuda").bfloat16()
    o_nh = torch.empty(n, h, dtype=torch.bfloat16, device="cuda")
    o_nd = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    o_hd = torch.empty(h, d, dtype=torch.bfloat16, device="cuda")
    o_dh = torch.empty(d, h, dtype=torch.bfloat16, device="cuda")

    def cublas_gemms():
        torch.matmul(x, w1, out=o_nh)           # fwd.pre_act   [n,d]x[d,h]
        torch.matmul(act, w2, out=o_nd)         # fwd.out       [n,h]x[h,d]
        torch.matmul(dy, w2.t(), out=o_nh)      # bwd.d_act     [n,d]x[d,h]
        torch.matmul(act.t(), dy, out=o_hd)     # bwd.d_w2      [h,n]x[n,d]
        torch.matmul(x.t(), g, out=o_dh)        # bwd.d_w1      [d,n]x[n,h]
        torch.matmul(g, w1.t(), out=o_nd)       # bwd.d_x       [n,h]x[h,d]

    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            cublas_gemms()
    torch.cuda.current_stream().wait_stream(st)
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        cublas_gemms()
    p = s24.FfnParams(w1=w1, w2=w2)
    graphs = {"cuBLAS six GEMMs": cg}
    for name, cfg in (("s24 dense twin step", s24.FfnConfig()), ("s24 recipe step", s24.RECIPE)):
        sg = s24.FfnStepGraph(p, cfg, n)
        sg.x.copy_(x)
        sg.dy.copy_(dy)
        graphs[name] = sg
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {k: [] for k in graphs}
    names = list(graphs)
    for b in range(args.blocks):
        for name in names[b % len(names):] + names[:b % len(names)]:  # (rotate the order per block)
            gr = graphs[name]
            evs = []
            for _ in range(args.steps):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                gr.replay()
                e.record()
                evs.append((s, e))
            torch.cuda.synchronize()
            res[name].append(statistics.median(s.elapsed_time(e) for s, e in evs))
    print(json.dumps({k: {"median_ms": round(statistics.median(v), 4), "min_ms": round(min(v), 4)}
                      for k, v in res.items()}))


if __name__ == "__main__":
    main()
