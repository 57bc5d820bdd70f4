"""Toy-scale recipe parity (ref tests/test_acceptance.py:294-318, SURVEY 8f
row 1): a byte-level LM whose FFN blocks run on the B200 kernels trains to
the same eval loss with the full recipe (dense warmup, sparse24 forward,
split backward, plans reused for 2 steps) as with the dense FFN, within the
reference's 5% gap; plus the harness API (metrics, ablation rows, divergence,
checkpoints)."""

import json
import math
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from paper_2503_16672_b200 import toy

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def corpus() -> bytes:
    files = ["DESIGN.md", "INTEGRATION.md", "paper_2503_16672_b200/ffn.py", "paper_2503_16672_b200/splitgemm.py",
             "oracle/srelu24_np.py", "bench.py"]
    return b"\n".join((ROOT / f).read_bytes() for f in files)


def test_recipe_trains_like_dense(tmp_path):
    path = tmp_path / "corpus.txt"
    path.write_bytes(corpus())
    mc = toy.ToyModelConfig(embed_dim=64, hidden=256, num_blocks=2, context=8)
    tc = toy.TrainConfig(steps=400, warmup_dense_steps=40, batch_tokens=256, lr=3e-3, lr_warmup_steps=40,
                         eval_every=200, eval_tokens=4096, plan_refresh_every=2)
    rows = {r.key: r for r in toy.ablate(path, mc, tc, rows=("dense-relu2", "recipe"))}
    dense, recipe = rows["dense-relu2"], rows["recipe"]
    assert not dense.diverged and not recipe.diverged
    assert math.isfinite(recipe.final_eval_loss) and recipe.final_eval_loss < 3.5  # learned (ln 256 = 5.5)
    gap = abs(recipe.final_eval_loss - dense.final_eval_loss) / dense.final_eval_loss
    assert gap <= 0.05, (recipe.final_eval_loss, dense.final_eval_loss)
    assert recipe.gemms_sparse_last_step > 0 and dense.gemms_sparse_last_step == 0
    print(f"[reported] eval dense {dense.final_eval_loss:.4f} recipe {recipe.final_eval_loss:.4f} gap {gap:.2%}")


def test_harness_metrics_checkpoint_and_divergence(tmp_path):
    mc = toy.ToyModelConfig(embed_dim=64, hidden=128, num_blocks=2, context=8)
    tc = toy.TrainConfig(steps=20, warmup_dense_steps=5, batch_tokens=128, lr_warmup_steps=5, eval_every=10,
                         eval_tokens=512, ffn=s24.RECIPE)
    metrics, model = toy.train(mc, tc, corpus())
    assert [m.step for m in metrics] == [10, 20]
    last = metrics[-1]
    assert len(last.per_layer_sparsity) == 2 and all(0.0 <= s <= 1.0 for s in last.per_layer_sparsity)
    assert all(0.0 <= f < 1.0 for f in last.per_layer_dropped_fraction)
    # recipe census per block: fwd.pre_act (dense), fwd.out (2:4), bwd.d_act (dense), dW2, dW1, dX (2:4)
    assert last.gemms_dense == 2 * 2 and last.gemms_sparse == 2 * 4 and last.macs_this_step > 0
    csv = toy.metrics_to_csv(metrics).splitlines()
    assert csv[0] == toy.METRICS_HEADER and len(csv) == 1 + 2 * 2
    toy.save_checkpoint(tmp_path / "ckpt", model, mc, tc, 20, corpus="corpus.txt")
    man = json.loads((tmp_path / "ckpt" / "manifest.json").read_text())
    assert man["step"] == 20 and set(man["params"]) == set(model.param_dict())
    w = s24.read_matrix(tmp_path / "ckpt" / man["params"]["block0.w1"]["file"])
    assert np.array_equal(w, model.w1[0].detach().cpu().numpy())

    def blow_up(step, grads):  # a NaN gradient at step 3 is reported with its step
        if step == 3:
            grads = dict(grads)
            grads["head"] = torch.full_like(grads["head"], float("nan"))
        return grads

    with pytest.raises(s24.DivergenceError) as ei:
        toy.train(mc, tc, corpus(), grad_transform=blow_up)
    assert ei.value.step == 3
    with pytest.raises(s24.ConfigError):
        toy.ablate(corpus(), mc, tc, rows=["dense-swiglu"])


def test_init_activation_sparsity_is_about_half():
    """ref tests/test_acceptance.py:107-122 (c03): at initialisation about half
    of the squared-ReLU activations are zero, per layer."""
    mc = toy.ToyModelConfig(embed_dim=64, hidden=256, num_blocks=2, context=8)
    train_split, _ = toy.build_dataset(corpus(), mc.context, 0.9)
    model = toy.ToyModel(mc)
    sp = toy.measure_activation_sparsity(model, train_split.contexts[:2048])
    assert len(sp) == 2 and all(abs(s - 0.5) <= 0.05 for s in sp), sp


def test_untileable_dims_train():
    """embed_dim 24, hidden 100: the FFN blocks run zero-padded (ffn.ffn_forward)."""
    mc = toy.ToyModelConfig(embed_dim=24, hidden=100, num_blocks=2, context=8)
    tc = toy.TrainConfig(steps=12, warmup_dense_steps=4, batch_tokens=64, lr_warmup_steps=4, eval_every=6,
                         eval_tokens=256, ffn=s24.RECIPE)
    metrics, model = toy.train(mc, tc, corpus())
    assert [m.step for m in metrics] == [6, 12]
    assert all(np.isfinite(m.eval_loss) for m in metrics)
    assert model.w1[0].shape == (24, 100)
    assert metrics[-1].gemms_sparse == 2 * 4
