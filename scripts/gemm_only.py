"""Run one fused GEMM (K1 / K3 / dense dact / sparse fwd) alone at the c2 shape, for profiling."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
which = sys.argv[1]
n, d, h = (16384, 2048, 8192) if len(sys.argv) < 3 else tuple(int(v) for v in sys.argv[2:5])
S = torch.cuda.current_stream().cuda_stream
bf = torch.bfloat16
x = torch.randn(n, d, device="cuda", dtype=bf)
w1 = (torch.randn(d, h, device="cuda") / d**0.5).to(bf)
w2 = (torch.randn(h, d, device="cuda") / h**0.5).to(bf)
vals = torch.zeros(n, h // 2, device="cuda", dtype=bf)
meta = torch.full((_lib.meta_hw_bytes(n, h),), 0x44, device="cuda", dtype=torch.uint8)
counts = torch.zeros(h, device="cuda", dtype=torch.int32)
stats = torch.zeros(2, device="cuda", dtype=torch.int64)
act = torch.empty(n, h, device="cuda", dtype=bf)
gv = torch.empty_like(vals)
out = torch.empty(n, d, device="cuda", dtype=bf)
_lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(vals), P(meta), P(counts), P(stats), None, None, None, None, 0, None, S)
for _ in range(4):
    if which == "k1":
        _lib.call("s24_fwd_gemm1_fused", P(x), d, P(w1), h, n, h, d, P(vals), P(meta), P(counts), P(stats), None, None, None, None, 0, None, S)
    elif which == "k3":
        _lib.call("s24_bwd_dact_fused", P(x), d, P(w2), d, n, h, d, P(vals), P(meta), P(gv), None, None, None, 0, None, S)
    elif which == "dact":
        _lib.call("s24_gemm_dact", P(x), d, P(w2), d, n, h, d, P(act), h, P(act), h, S)
    elif which == "relu2":
        _lib.call("s24_gemm_relu2", P(x), d, P(w1), h, n, h, d, P(act), h, S)
    elif which == "spfwd":
        _lib.call("s24_spmm", P(vals), P(meta), P(w2), 1, d, n, d, h, P(out), 1, d, None, 0, -1, None, 0, S)
torch.cuda.synchronize()
print("ok", which)
