"""One plain dense GEMM of ours and one cuBLAS GEMM at the K1 shape (c2:
16384 x 8192 x 2048, bf16 out), for an ncu side-by-side."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: None if t is None else t.data_ptr()  # noqa: E731
n, d, h = (16384, 2048, 8192) if len(sys.argv) < 4 else tuple(int(v) for v in sys.argv[1:4])
bf = torch.bfloat16
x = torch.randn(n, d, device="cuda", dtype=bf)
w1 = (torch.randn(d, h, device="cuda") / d**0.5).to(bf)
act = torch.empty(n, h, device="cuda", dtype=bf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
S = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    flush.zero_()
    _lib.call("s24_gemm", P(x), 0, d, P(w1), 1, h, n, h, d, P(act), 1, h, None, 0, -1, None, S)
    flush.zero_()
    torch.matmul(x, w1, out=act)
torch.cuda.synchronize()
print("ok")
