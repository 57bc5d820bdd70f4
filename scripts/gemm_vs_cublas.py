"""Plain bf16 GEMMs (bf16 out, fp32 accumulation) of the c2 step's shapes:
this repo's engine (s24_gemm, no epilogue work) against cuBLAS
(torch.matmul), each shape captured in a CUDA graph of `--reps` launches, the
two implementations alternated over `--blocks` blocks.

usage: python scripts/gemm_vs_cublas.py [--n 16384 --d 2048 --h 8192] [--reps 10] [--blocks 6]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--h", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--blocks", type=int, default=6)
    args = ap.parse_args()
    n, d, h = args.n, args.d, args.h
    r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
    x, w1, w2, dy, act, g = r(n, d), r(d, h), r(h, d), r(n, d), r(n, h), r(n, h)
    o_nh, o_nd = torch.empty(n, h, dtype=torch.bfloat16, device="cuda"), torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    P = lambda t: t.data_ptr()  # noqa: E731
    S = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    BF = 1
    shapes = {
        # name: (cuBLAS call, s24 call) ; s24_gemm(A, a_mn, lda, B, b_mn, ldb, M, N, K, D, dtype, ldd, ...)
        "pre_act [n,d]x[d,h]": (lambda: torch.matmul(x, w1, out=o_nh),
                                lambda: _lib.call("s24_gemm", P(x), 0, d, P(w1), 1, h, n, h, d, P(o_nh), BF, h, None, 0, -1, None, S())),
        "d_act [n,d]x[h,d]^T": (lambda: torch.matmul(dy, w2.t(), out=o_nh),
                                lambda: _lib.call("s24_gemm", P(dy), 0, d, P(w2), 0, d, n, h, d, P(o_nh), BF, h, None, 0, -1, None, S())),
        "fwd.out dense [n,h]x[h,d]": (lambda: torch.matmul(act, w2, out=o_nd),
                                      lambda: _lib.call("s24_gemm", P(act), 0, h, P(w2), 1, d, n, d, h, P(o_nd), BF, d, None, 0, -1, None, S())),
        "d_x dense [n,h]x[d,h]^T": (lambda: torch.matmul(g, w1.t(), out=o_nd),
                                    lambda: _lib.call("s24_gemm", P(g), 0, h, P(w1), 0, h, n, d, h, P(o_nd), BF, d, None, 0, -1, None, S())),
    }

    def graph(fn):
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            fn()
        torch.cuda.current_stream().wait_stream(st)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(args.reps):
                fn()
        return gr

    graphs = {(k, impl): graph(fns[i]) for k, fns in shapes.items() for i, impl in enumerate(("cublas", "s24"))}
    res = {key: [] for key in graphs}
    for _ in range(args.blocks):
        for key, gr in graphs.items():
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            gr.replay()
            e.record()
            torch.cuda.synchronize()
            res[key].append(s.elapsed_time(e) / args.reps * 1e3)
    out = {}
    for k in shapes:
        c, o = statistics.median(res[(k, "cublas")]), statistics.median(res[(k, "s24")])
        out[k] = {"cublas_us": round(c, 1), "s24_us": round(o, 1), "s24_over_cublas": round(o / c, 3)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
