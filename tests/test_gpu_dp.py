"""Token-sharding parity on one GPU: what each rank of the
data-parallel run computes, checked against the unsharded run and the oracle.

* prefill: the concatenated per-shard outputs equal the single-GPU output bit
  for bit (every stage maps one token row to one output row; the permutation
  only reorders rows);
* training: each shard runs the recipe with its own permutation and plan (the
  reference applied per shard), so dW = sum over shards of the per-shard
  oracle, within the bf16 tolerance; dX per shard is the unsharded kernel's
  result on that shard.
"""

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from oracle import srelu24_np as O
from paper_2503_16672_b200 import dp

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("fp8", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_prefill_shards_concatenate_bitwise(world, fp8):
    # (e4m3: per-token scales and shared weight codes keep rows independent)
    n, d, h = 1536, 256, 512
    x, w1, w2, _ = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=41)
    p = s24.FfnParams(w1=w1, w2=w2)
    tx = torch.from_numpy(x).cuda().bfloat16()
    cfg = s24.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
                        permute_tokens=False, fp8_emulation=fp8)
    full, _ = s24.ffn_forward(tx, p, cfg, for_backward=False)
    parts = []
    for r in range(world):
        a, b = dp.shard_bounds(n, world, r)
        parts.append(dp.prefill(tx[a:b], p, cfg))
    assert torch.equal(torch.cat(parts), full)


@pytest.mark.parametrize("fp8", [False, True])
def test_training_shards_sum_to_per_shard_reference(fp8):
    """fp8=True: the e4m3 recipe (fp8_emulation + fp8_backward) per shard vs
    the oracle's emulation per shard (tolerances as in test_gpu_ffn_fp8)."""
    n, d, h, world = 1024, 256, 512, 2
    x, w1, w2, dy = O.synthetic_ffn_inputs(n, d, h, sparsity=0.9, seed=43)
    xb, w1b, w2b, dyb = (O.bf16_round(t) for t in (x, w1, w2, dy))
    p = s24.FfnParams(w1=w1, w2=w2)
    cfg = s24.RECIPE
    ocfg = O.RECIPE
    tol_o, tol_g, tol_w = 1e-2, 1e-2, 8e-3
    if fp8:
        from dataclasses import replace

        cfg = replace(cfg, fp8_emulation=True, fp8_backward=True)
        ocfg = dict(ocfg, fp8_emulation=True, fp8_backward=True)
        tol_o, tol_g, tol_w = 1e-2, 3e-2, 3e-2
    dw1 = np.zeros((d, h))
    dw2 = np.zeros((h, d))
    ref_dw1 = np.zeros((d, h))
    ref_dw2 = np.zeros((h, d))
    for r in range(world):
        a, b = dp.shard_bounds(n, world, r)
        tx = torch.from_numpy(xb[a:b]).cuda().bfloat16()
        tg = torch.from_numpy(dyb[a:b]).cuda().bfloat16()
        out, cache = s24.ffn_forward(tx, p, cfg)
        g = s24.ffn_backward(tg, cache, p, cfg)
        dw1 += g.d_w1.double().cpu().numpy()
        dw2 += g.d_w2.double().cpu().numpy()
        o_out, o_cache = O.ffn_forward(xb[a:b], w1b, w2b, ocfg, ordered=False)
        o_g = O.ffn_backward(dyb[a:b], o_cache, w1b, w2b, ocfg, ordered=False)
        ref_dw1 += o_g["d_w1"]
        ref_dw2 += o_g["d_w2"]
        assert rel(out.float().cpu().numpy(), o_out) < tol_o
        assert rel(g.d_x.float().cpu().numpy(), o_g["d_x"]) < tol_g
    assert rel(dw1, ref_dw1) < tol_w
    assert rel(dw2, ref_dw2) < tol_w
