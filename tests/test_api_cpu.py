"""Host-side logic of the drop-in API that needs no GPU: config validation
(ref tests/test_ffn.py:85-114), split-plan sizing, MAC accounting, token
sharding, and the loud failure when no device is present."""

import numpy as np
import pytest
import torch

import paper_2503_16672_b200 as s24
from paper_2503_16672_b200.dp import shard_bounds
from paper_2503_16672_b200.splitgemm import ceil_fraction


def test_config_defaults_and_recipe():
    c = s24.FfnConfig()
    assert (c.forward_mode, c.backward_mode, c.split_ratio) == ("dense", "dense", 0.95)
    r = s24.RECIPE
    assert r.forward_mode == "sparse24" and r.backward_mode == "split_masked"
    assert r.mask_grad_with_fwd and r.permute_tokens
    d = r.densified()
    assert d.forward_mode == "dense" and not d.permute_tokens and d.split_ratio == r.split_ratio


@pytest.mark.parametrize("kw", [
    dict(backward_mode="split_masked"),
    dict(backward_mode="naive_sparse"),
    dict(mask_grad_with_fwd=True),
    dict(split_ratio=1.5),
    dict(split_ratio=-0.1),
    dict(fp8_backward=True),
    dict(activation="gelu"),
    dict(forward_mode="sparse"),
    dict(backward_mode="weird"),
    dict(activation="swiglu", forward_mode="sparse24"),
])
def test_config_validation(kw):
    with pytest.raises(s24.ConfigError):
        s24.FfnConfig(**kw)


def test_ceil_fraction_matches_reference_cases():
    # ref tests/test_splitgemm.py:57-59 and the float-noise guard (splitgemm.py:33-38)
    assert ceil_fraction(0.95, 4096) == 3892
    assert ceil_fraction(0.95, 16384) == 15565
    assert ceil_fraction(0.95, 8192) == 7783
    assert ceil_fraction(0.29, 100) == 29
    assert ceil_fraction(0.5, 3) == 2


def test_mac_accounting():
    assert s24.gemm_macs(2, 3, 4) == 24
    assert s24.sp_gemm_macs(4, 8, 2) == 32


def test_token_shards_cover_and_align():
    for n, g in [(16384, 8), (32768, 3), (4096, 1), (100, 7)]:
        bounds = [shard_bounds(n, g, r) for r in range(g)]
        assert bounds[0][0] == 0 and bounds[-1][1] == n
        for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
            assert a1 == b0
        assert all((b - a) % 4 == 0 for a, b in bounds)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 0)


def test_permutation_is_the_reference_stream():
    # PCG64 Fisher-Yates from the top: same as ref matcore.py:269-280
    p = s24.make_permutation(0, 16)
    assert sorted(p.tolist()) == list(range(16))
    assert np.array_equal(p, s24.make_permutation(0, 16))
    assert not np.array_equal(p, s24.make_permutation(1, 16))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device failure mode")
def test_no_cpu_fallback():
    with pytest.raises(s24.BackendError):
        s24.sparsify_token_wise(np.zeros((4, 8), np.float32))
    with pytest.raises(s24.BackendError):
        s24.FfnParams(w1=np.zeros((8, 16), np.float32), w2=np.zeros((16, 8), np.float32))


def test_toy_schedule_and_config_validation():
    import math as _m

    from paper_2503_16672_b200 import toy
    from paper_2503_16672_b200.errors import ConfigError
    tc = toy.TrainConfig(steps=100, lr=1.0, lr_warmup_steps=10, warmup_dense_steps=5)
    assert toy.lr_at(tc, 5) == 0.5 and toy.lr_at(tc, 10) == 1.0
    assert toy.lr_at(tc, 11) == 1.0 and abs(toy.lr_at(tc, 100)) < 1e-12
    assert abs(toy.lr_at(tc, 55) - 0.5 * (1 + _m.cos(_m.pi * 44 / 89))) < 1e-12
    for bad in (dict(batch_tokens=0), dict(steps=10, warmup_dense_steps=11), dict(plan_refresh_every=0),
                dict(eval_every=0), dict(lr_schedule="step"), dict(split_fraction=0.0)):
        with pytest.raises(ConfigError):
            toy.TrainConfig(**bad)
    with pytest.raises(ConfigError):
        toy.ToyModelConfig(hidden=102)
    with pytest.raises(ConfigError):
        toy.ToyModelConfig(embed_dim=60, context=8)
    toy.ToyModelConfig(hidden=100, embed_dim=24)  # (run zero-padded on the device)
    tr, ev = toy.build_dataset(bytes(range(20)), 4, 0.5, "cpu")
    assert tr.contexts.shape == (8, 4) and ev.contexts.shape == (8, 4) and len(tr) == 8
    assert tr.contexts[3].tolist() == [3, 4, 5, 6] and int(tr.targets[3]) == 7
    from paper_2503_16672_b200.errors import DataError
    with pytest.raises(DataError):
        toy.build_dataset(b"abc", 4, 0.9, "cpu")
    assert [k for k, _ in toy.ABLATION_ROWS][:3] == ["dense-swiglu", "dense-relu2", "recipe"]
    mc, tcr = toy.ablation_configs(toy.ToyModelConfig(), toy.TrainConfig(), "no-permute")
    assert tcr.ffn.forward_mode == "sparse24" and not tcr.ffn.permute_tokens


def test_permutation_caches_are_bounded():
    """one cache entry per distinct token count must not grow
    without bound (LRU of _CACHE_ENTRIES)."""
    from paper_2503_16672_b200 import matcore as M

    for n in range(4, 4 + 4 * (M._CACHE_ENTRIES + 10), 4):
        p = M.make_permutation(0, n)
        assert sorted(p.tolist()) == list(range(n))
    assert len(M._perm_cache) == M._CACHE_ENTRIES
    again = M.make_permutation(0, 8)  # evicted long ago: recomputed, same stream
    assert again.tolist() == M.make_permutation(0, 8).tolist()
