"""Per-kernel timing at the bench shapes (CUDA events, warm, L2 flushed between
iterations). Prints one line per kernel: time, TFLOP/s (dense-equivalent),
fraction of measured peaks, and cuBLAS (torch.matmul) for the same GEMM shape.

usage: python scripts/kernel_bench.py [--config c2|c3] [--iters 10]
"""

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
S = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
CONFIGS = {"c1": (4096, 512, 2048), "c2": (16384, 2048, 8192), "c3": (32768, 4096, 16384)}


def timeit(fn, iters, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    n, d, h = CONFIGS[args.config]
    peaks = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text()) if (
        Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else {"bf16_tflops": 1643.4,
                                                                                        "hbm_gbs": 6545.9}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    torch.manual_seed(0)
    bf = torch.bfloat16
    x = torch.randn(n, d, device="cuda", dtype=bf)
    w1 = (torch.randn(d, h, device="cuda") / d**0.5).to(bf)
    w2 = (torch.randn(h, d, device="cuda") / h**0.5).to(bf)
    g = torch.randn(n, d, device="cuda", dtype=bf)
    act_vals = torch.zeros(n, h // 2, device="cuda", dtype=bf)
    meta = torch.zeros(_lib.meta_hw_bytes(n, h), device="cuda", dtype=torch.uint8)
    counts = torch.zeros(h, device="cuda", dtype=torch.int32)
    stats = torch.zeros(3, device="cuda", dtype=torch.int64)
    out = torch.empty(n, d, device="cuda", dtype=bf)
    act = torch.empty(n, h, device="cuda", dtype=bf)
    gv = torch.zeros_like(act_vals)
    rows = []

    def rec(name, ms, flops, cublas_ms=None, bytes_=None):
        tf = flops / ms / 1e9
        r = {"kernel": name, "ms": round(ms, 4), "tflops_dense_equiv": round(tf, 1),
             "frac_dense_peak": round(tf / peaks["bf16_tflops"], 3)}
        if cublas_ms:
            r["cublas_ms"] = round(cublas_ms, 4)
            r["vs_cublas"] = round(cublas_ms / ms, 3)
        if bytes_:
            r["GB/s"] = round(bytes_ / ms / 1e6, 1)
            r["frac_hbm"] = round(bytes_ / ms / 1e6 / peaks["hbm_gbs"], 3)
        rows.append(r)
        print(json.dumps(r), flush=True)

    f = 2.0 * n * d * h
    cb1 = timeit(lambda: torch.matmul(x, w1), args.iters, flush)
    rec("K1 fwd gemm1 fused", timeit(lambda: _lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(act_vals),
                                                          P(meta), P(counts), P(stats), None, S()), args.iters, flush),
        f, cb1)
    rec("dense relu2 (twin of K1)", timeit(lambda: _lib.call("s24_gemm_relu2", P(x), d, P(w1), h, n, h, d, P(act), h,
                                                                S()), args.iters, flush), f, cb1)
    rec("dense plain store (K1 shape)", timeit(lambda: _lib.call("s24_gemm", P(x), 0, d, P(w1), 1, h, n, h, d, P(act),
                                                                    1, h, None, 0, -1, None, S()), args.iters, flush),
        f, cb1)
    cb2 = timeit(lambda: torch.matmul(act, w2), args.iters, flush)
    rec("K2 fwd.out sparse", timeit(lambda: _lib.call("s24_spmm", P(act_vals), P(meta), P(w2), 1, d, n, d, h, P(out),
                                                         1, d, None, 0, -1, None, 0, S()), args.iters, flush), f, cb2)
    rec("fwd.out dense twin", timeit(lambda: _lib.call("s24_gemm", P(act), 0, h, P(w2), 1, d, n, d, h, P(out), 1, d,
                                                          None, 0, -1, None, S()), args.iters, flush), f, cb2)
    cb3 = timeit(lambda: torch.matmul(g, w2.t()), args.iters, flush)
    rec("K3 bwd dact fused", timeit(lambda: _lib.call("s24_bwd_dact_fused", P(g), d, P(w2), d, n, h, d, P(act_vals),
                                                         P(meta), P(gv), S()), args.iters, flush), f, cb3)
    rec("dense dact (twin of K3)", timeit(lambda: _lib.call("s24_gemm_dact", P(g), d, P(w2), d, n, h, d, P(act), h,
                                                               P(act), h, S()), args.iters, flush), f, cb3)
    cb4 = timeit(lambda: torch.matmul(act, w1.t()), args.iters, flush)
    rec("K2 bwd.d_x sparse", timeit(lambda: _lib.call("s24_spmm", P(gv), P(meta), P(w1), 0, h, n, d, h, P(out), 1, d,
                                                         None, 0, -1, None, 0, S()), args.iters, flush), f, cb4)
    rec("bwd.d_x dense twin", timeit(lambda: _lib.call("s24_gemm", P(act), 0, h, P(w1), 0, h, n, d, h, P(out), 1, d,
                                                          None, 0, -1, None, S()), args.iters, flush), f, cb4)
    dw = torch.empty(h, d, device="cuda")
    cb5 = timeit(lambda: torch.matmul(act.t(), g), args.iters, flush)
    rec("bwd.d_w dense twin (A MN)", timeit(lambda: _lib.call("s24_gemm", P(act), 1, h, P(g), 1, d, h, d, n, P(dw), 0,
                                                                 d, None, 0, -1, None, S()), args.iters, flush), f, cb5)
    ns = (int(0.95 * h) + 127) // 128 * 128
    vs = torch.zeros(ns, n // 2, device="cuda", dtype=bf)
    es = torch.full((_lib.meta_hw_bytes(ns, n),), 0x44, device="cuda", dtype=torch.uint8)
    rec("bwd.d_w sparse part (M=0.95h)", timeit(lambda: _lib.call("s24_spmm", P(vs), P(es), P(g), 1, d, ns, d, n,
                                                                     P(dw), 0, d, None, 0, -1, None, 0, S()), args.iters, flush),
        2.0 * ns * d * n)
    # K4 split
    kcount = int(0.95 * h)
    pos = torch.empty(h, dtype=torch.int32, device="cuda")
    sp = torch.empty(h, dtype=torch.int32, device="cuda")
    de = torch.empty(h, dtype=torch.int32, device="cuda")
    counts.copy_(torch.randint(0, n, (h,), device="cuda", dtype=torch.int32))
    rec("K7 plan", timeit(lambda: _lib.call("s24_plan", P(counts), h, kcount, P(sp), P(de), P(pos), S()), args.iters,
                          flush), 0.0 + 1e-9)
    vd = torch.zeros((h - kcount + 127) // 128 * 128, n, device="cuda", dtype=bf)
    k4_bytes = n * h * 1.125 + kcount * n * 1.125 + (h - kcount) * n * 2
    rec("K4 feature split", timeit(lambda: _lib.call("s24_feature_split", P(act_vals), P(meta), n, h, P(pos), kcount,
                                                        h - kcount, P(vs), P(es), P(vd), P(stats), 1, -1, S()), args.iters,
                                    flush), 1e-9, bytes_=k4_bytes)
    nd = h - kcount
    vsx = torch.empty((2 * nd + kcount + 127) // 128 * 128 + 1, n // 2, device="cuda", dtype=bf)
    esx = torch.empty(_lib.meta_hw_bytes((2 * nd + kcount + 127) // 128 * 128 + 128, n), device="cuda",
                      dtype=torch.uint8)
    k4x_bytes = n * h * 1.125 + (2 * nd + kcount) * n * 0.5625
    rec("K4x paired (hot path)", timeit(lambda: _lib.call("s24_feature_split_x", P(act_vals), P(meta), n, h,
                                                             P(pos), kcount, nd, P(vsx), P(esx), 1, None, S()),
                                         args.iters, flush), 1e-9, bytes_=k4x_bytes)
    src = torch.randperm(n, device="cuda").int()
    rec("K6 gather rows", timeit(lambda: _lib.call("s24_gather_rows", P(x), n, 2 * d, 2 * d, P(src), P(out), 2 * d,
                                                      S()), args.iters, flush), 1e-9, bytes_=2 * n * d * 2)


if __name__ == "__main__":
    main()
