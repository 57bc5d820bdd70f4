"""dW grouped 2:4 GEMM at the c2 shape (M = 8601 paired rows, N = 2048,
K = 16384 tokens) under raster group heights S24_GROUP_M (interleaved
rounds, L2 flushed, CUDA events)."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
S = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
M, N, K = 8601, 2048, 16384
mp = (M + 127) // 128 * 128
bf = torch.bfloat16
ops = []
for _ in range(2):
    vs = torch.randn(mp, K // 2, device="cuda").to(bf)
    es = torch.full((_lib.meta_hw_bytes(mp, K),), 0x44, dtype=torch.uint8, device="cuda")
    b = torch.randn(K, N, device="cuda").to(bf)
    ops.append((vs, es, b))
out0 = torch.empty(M, N, device="cuda")
out1 = torch.empty(N, M, device="cuda")
rmap = torch.arange(M, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
(v0, e0, b0), (v1, e1, b1) = ops


def run():
    _lib.call("s24_spmm_pair", 1, M, N, K, 0, P(v0), P(e0), P(b0), N, P(out0), N, P(rmap), 0, None,
              P(v1), P(e1), P(b1), N, P(out1), M, P(rmap), 1, None, 818, S())


res = {}
for rnd in range(4):
    for gm in ("2", "4", "6", "8", "12"):
        os.environ["S24_GROUP_M"] = gm
        for _ in range(2):
            run()
        ts = []
        for _ in range(5):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run()
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        res.setdefault(gm, []).extend(ts)
for gm, v in res.items():
    print(f"group_m={gm:>3}: median {statistics.median(v):.4f} ms  min {min(v):.4f}")
