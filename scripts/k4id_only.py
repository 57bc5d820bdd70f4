"""Run the identity-layout K4 alone at the c2 shape (profiling)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: t.data_ptr()  # noqa: E731
n, h = 16384, 8192
S = torch.cuda.current_stream().cuda_stream
a = torch.relu(torch.randn(n, h, device="cuda")).square().bfloat16()
vals = torch.zeros(n, h // 2, device="cuda", dtype=torch.bfloat16)
meta = torch.zeros(_lib.meta_hw_bytes(n, h), device="cuda", dtype=torch.uint8)
_lib.call("s24_sparsify_token", P(a), 1, n, h, h, P(vals), None, P(meta), None, None, S)
ks = int(0.95 * h)
counts = torch.randint(0, n, (h,), device="cuda", dtype=torch.int32)
pos = torch.empty(h, dtype=torch.int32, device="cuda")
sp = torch.empty(h, dtype=torch.int32, device="cuda")
de = torch.empty(h, dtype=torch.int32, device="cuda")
_lib.call("s24_plan", P(counts), h, ks, P(sp), P(de), P(pos), S)
nd = h - ks
pad = (2 * nd + 127) // 128 * 128
vs = torch.empty(pad + h, n // 2, device="cuda", dtype=torch.bfloat16)
es = torch.empty(_lib.meta_hw_bytes(pad + h, n), device="cuda", dtype=torch.uint8)
for _ in range(5):
    _lib.call("s24_feature_split_id", P(vals), P(meta), n, h, P(pos), nd, P(vs), P(es), None, 1, S)
torch.cuda.synchronize()
print("ok")
