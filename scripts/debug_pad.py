"""Scratch: d_w2 error vs the oracle for a few (n, d, h) in naive_sparse mode."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


cfg = s24.FfnConfig(forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True)
cd = dict(forward_mode=cfg.forward_mode, backward_mode=cfg.backward_mode, mask_grad_with_fwd=True,
          permute_tokens=False, permute_seed=0, split_ratio=0.95)
for (n, d, h, seed) in [(64, 48, 200, 312), (64, 64, 256, 312), (64, 48, 200, 5), (64, 64, 256, 5), (192, 48, 200, 312),
                        (128, 48, 200, 312), (60, 48, 200, 312), (64, 48, 256, 312), (64, 64, 200, 312)]:
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.8, seed=seed)
    p = s24.FfnParams(w1=torch.from_numpy(w1).cuda(), w2=torch.from_numpy(w2).cuda())
    out, cache = s24.ffn_forward(torch.from_numpy(x).cuda(), p, cfg, keep_pre_act=True)
    g = s24.ffn_backward(torch.from_numpy(dy).cuda(), cache, p, cfg)
    torch.cuda.synchronize()
    oo, oc = O.ffn_forward(x, w1, w2, cd, ordered=False)
    og = O.ffn_backward(dy, oc, w1, w2, cd, ordered=False)
    dev_act = s24.decompress(cache.act_sparse).cpu().numpy()
    flips = int((oc["mask"] != cache.fwd_mask.cpu().numpy()).sum())
    # d_w2 from the device's own act, oracle feature selection
    v, m, _, _ = O.sparsify_feature(dev_act)
    w2_replay = O.gemm_at(O.decompress_feature(v, m, *dev_act.shape), dy, False)
    print(n, d, h, seed, "flips", flips, "out", f"{rel(out.float().cpu(), oo):.2e}", "dw2", f"{rel(g.d_w2.cpu(), og['d_w2']):.2e}",
          "dw2 replay", f"{rel(g.d_w2.cpu(), w2_replay):.2e}", "dw1", f"{rel(g.d_w1.cpu(), og['d_w1']):.2e}",
          "act", f"{rel(dev_act, oc['act']):.2e}", flush=True)
