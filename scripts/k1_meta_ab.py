"""K1 (s24_fwd_gemm1_fused) at c2, interleaved A/B: no row map (metadata
gathered across lane pairs, 16-byte stores) vs an identity row map (per-chunk
2-byte metadata stores). L2 flushed between launches, CUDA events."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
n, d, h = 16384, 2048, 8192
bf = torch.bfloat16
x = torch.randn(n, d, device="cuda", dtype=bf)
w1 = (torch.randn(d, h, device="cuda") / d**0.5).to(bf)
vals = torch.zeros(n, h // 2, device="cuda", dtype=bf)
meta_a = torch.zeros(_lib.meta_hw_bytes(n, h), device="cuda", dtype=torch.uint8)
meta_b = torch.zeros_like(meta_a)
counts = torch.zeros(h, device="cuda", dtype=torch.int32)
stats = torch.zeros(2, device="cuda", dtype=torch.int64)
ident = torch.arange(n, device="cuda", dtype=torch.int32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S = torch.cuda.current_stream().cuda_stream


def k1(meta, rmap):
    _lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(vals), P(meta), P(counts), P(stats), None, None,
              None, None, 0, P(rmap), S)


def t(fn):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for _ in range(3):
    k1(meta_a, None)
    k1(meta_b, ident)
ta, tb = [], []
for _ in range(30):
    ta.append(t(lambda: k1(meta_a, None)))
    tb.append(t(lambda: k1(meta_b, ident)))
torch.cuda.synchronize()
print(f"combined meta {statistics.median(ta):.4f} ms  per-chunk meta {statistics.median(tb):.4f} ms  "
      f"identical metadata: {torch.equal(meta_a, meta_b)}")
