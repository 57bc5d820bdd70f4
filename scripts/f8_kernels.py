"""e4m3 kernel timings at the c2 shapes: plain dense e4m3 GEMM (K1 shape, bf16
out) vs the fused K1 / K3 e4m3 variants, the e4m3 2:4 GEMM, and cuBLAS-free
bf16 references (L2 flushed, CUDA events, median)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
S = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
n, d, h = 16384, 2048, 8192
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, iters=10):
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


def codes(*shape):
    c = torch.randint(0, 0x70, shape, dtype=torch.uint8, device="cuda")
    return c


xq, w1q, w2q = codes(n, d), codes(h, d), codes(h, d)
sx, s1, s2 = (torch.rand(k, device="cuda") + 0.5 for k in (n, h, h))
out_bf = torch.empty(n, h, dtype=torch.bfloat16, device="cuda")
vals32 = torch.empty(n, h // 2, device="cuda")
amax = torch.zeros(n, dtype=torch.int32, device="cuda")
meta = torch.full((_lib.meta_hw_bytes(n, h),), 0x44, dtype=torch.uint8, device="cuda")
counts = torch.zeros(h, dtype=torch.int32, device="cuda")
stats = torch.zeros(2, dtype=torch.int64, device="cuda")
act = torch.rand(n, h // 2, device="cuda").bfloat16()
gv = torch.empty_like(act)
fl = 2.0 * n * d * h
r = {}
r["gemm_f8 plain (K1 shape, bf16 out)"] = timeit(lambda: _lib.call("s24_gemm_f8", P(xq), d, P(w1q), d, n, h, d, P(sx), P(s1), P(out_bf), 1, h, None, 0, -1, S()))
r["K1 e4m3 fused"] = timeit(lambda: _lib.call("s24_fwd_gemm1_f8", P(xq), d, P(w1q), d, n, h, d, P(sx), P(s1), P(vals32), P(amax), P(meta), P(counts), P(stats), None, S()))
r["K3 e4m3 fused"] = timeit(lambda: _lib.call("s24_bwd_dact_f8", P(xq), d, P(w2q), d, n, h, d, P(sx), P(s2), P(act), P(meta), P(gv), S()))
for k, v in r.items():
    print(f"{v:8.4f} ms  {fl / v / 1e9:8.1f} TF/s  {k}")
