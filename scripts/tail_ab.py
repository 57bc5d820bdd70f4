"""Grouped dW 2:4 launch at the c2 shape (2 x M=8601, N=2048, K=16384, fp32
out), interleaved A/B: tail split on (default) vs S24_TAIL_SPLIT=0.
L2 flushed between launches, CUDA events, median of 20."""
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
M, N, K = 8601, 2048, 16384
mp = (M + 127) // 128 * 128
bf = torch.bfloat16
ops = []
for _ in range(2):
    v = (torch.randn(mp, K // 2, device="cuda") * 0.1).to(bf)
    e = torch.full((_lib.meta_hw_bytes(M, K),), 0x44, dtype=torch.uint8, device="cuda")
    b = torch.randn(K, N, device="cuda").to(bf)
    o = torch.empty(M, N, device="cuda")
    ops.append((v, e, b, o))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S = torch.cuda.current_stream().cuda_stream
(v0, e0, b0, o0), (v1, e1, b1, o1) = ops


def launch():
    _lib.call("s24_spmm_pair", 1, M, N, K, 0, P(v0), P(e0), P(b0), N, P(o0), N, None, 0, None,
              P(v1), P(e1), P(b1), N, P(o1), N, None, 0, None, 0, S)


def t(mode):
    os.environ["S24_TAIL_SPLIT"] = mode
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    launch()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for m in ("1", "0", "1", "0"):
    t(m)
on, off = [], []
for _ in range(20):
    on.append(t("1"))
    off.append(t("0"))
flops = 2 * 2 * M * N * K / 2
print(f"tail split {statistics.median(on):.4f} ms ({flops / statistics.median(on) / 1e9:.0f} TF/s dense-eq x2) | "
      f"without {statistics.median(off):.4f} ms")
