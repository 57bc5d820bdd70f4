"""A small recipe step (and its dense twin, the e4m3 variant and the API
sparsifiers) for compute-sanitizer: every hot-path kernel launches at least
once on a shape with ragged edges (n not a multiple of 256, d = 96 not a
multiple of the 256-wide tiles)."""
import sys
from dataclasses import replace
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2503_16672_b200 as s24  # noqa: E402
from oracle import srelu24_np as O  # noqa: E402

n, d, h = 640, 96, 384
x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=3)
p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
tx, tg = torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda()
for cfg in (s24.RECIPE, s24.FfnConfig(), replace(s24.RECIPE, fp8_emulation=True, fp8_backward=True)):
    out, cache = s24.ffn_forward(tx, p, cfg)
    g = s24.ffn_backward(tg, cache, p, cfg)
a = torch.randn(256, 512, device="cuda")
s24.sparsify_token_wise(a)
s24.sparsify_feature_wise_masked(a, torch.rand(256, 512, device="cuda") < 0.5)
torch.cuda.synchronize()
print("ok")
