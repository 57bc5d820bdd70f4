"""A few eager fp8 recipe steps at c2 (e4m3 forward + backward), for ncu captures."""
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2503_16672_b200 as s24  # noqa: E402

n, d, h = bench.CONFIGS["c2"]
x, w1, w2, dy = bench.synthetic_device_inputs(torch, n, d, h, seed=1234, device=torch.device("cuda"))
p = s24.FfnParams(w1=w1, w2=w2)
cfg = replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True)
for _ in range(3):
    out, cache = s24.ffn_forward(x, p, cfg)
    s24.ffn_backward(dy, cache, p, cfg)
torch.cuda.synchronize()
print("ok")
