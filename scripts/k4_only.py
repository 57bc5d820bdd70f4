"""Run K4 (feature split) alone at a bench shape, for profiling."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_16672_b200 import _lib  # noqa: E402

P = lambda t: t.data_ptr()  # noqa: E731
n, h = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 and sys.argv[1].isdigit() else (16384, 8192)
S = torch.cuda.current_stream().cuda_stream
a = torch.relu(torch.randn(n, h, device="cuda")).square().bfloat16()  # relu^2-like operand
vals = torch.zeros(n, h // 2, device="cuda", dtype=torch.bfloat16)
meta = torch.zeros(_lib.meta_hw_bytes(n, h), device="cuda", dtype=torch.uint8)
_lib.call("s24_sparsify_token", P(a), 1, n, h, h, P(vals), None, P(meta), None, None, S)
ks = int(0.95 * h)
counts = torch.randint(0, n, (h,), device="cuda", dtype=torch.int32)
pos = torch.empty(h, dtype=torch.int32, device="cuda")
sp = torch.empty(h, dtype=torch.int32, device="cuda")
de = torch.empty(h, dtype=torch.int32, device="cuda")
_lib.call("s24_plan", P(counts), h, ks, P(sp), P(de), P(pos), S)
vs = torch.zeros((ks + 127) // 128 * 128, n // 2, device="cuda", dtype=torch.bfloat16)
es = torch.zeros(_lib.meta_hw_bytes(ks, n), device="cuda", dtype=torch.uint8)
vd = torch.zeros((h - ks + 127) // 128 * 128, n, device="cuda", dtype=torch.bfloat16)
st = torch.zeros(2, dtype=torch.int64, device="cuda")
nd = h - ks
vsx = torch.zeros((2 * nd + ks + 127) // 128 * 128 + 1, n // 2, device="cuda", dtype=torch.bfloat16)
esx = torch.zeros(_lib.meta_hw_bytes((2 * nd + ks + 127) // 128 * 128 + 128, n), device="cuda", dtype=torch.uint8)
for _ in range(5):
    if "x" in sys.argv[3:]:  # the hot-path K4x (paired rank layout)
        _lib.call("s24_feature_split_x", P(vals), None, P(meta), n, h, P(pos), ks, nd, P(vsx), P(esx), None, None, 1, None, S)
    else:
        _lib.call("s24_feature_split", P(vals), P(meta), n, h, P(pos), ks, nd, P(vs), P(es), P(vd), None, 1, -1, S)
torch.cuda.synchronize()
print("ok")
