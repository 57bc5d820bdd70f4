"""TEST INFRASTRUCTURE ONLY -- regenerate tests/golden/*.npz from the reference.

Imports the reference implementation itself (pure Python/numpy, read-only at
/root/reference/pkg/src) and records its outputs on seeded inputs: the known
answer cases of the reference's own tests plus random cases for every
hot-path function (sparsifiers, mask compression, split plan, permutation,
split GEMM, full FFN forward/backward under several configs). The fixtures
are committed; /root/reference is not needed at test time.

usage: python oracle/make_golden.py [--ref /root/reference/pkg/src]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def bern(r, rows, cols, p):
    return ((r.random((rows, cols)) < p) * r.standard_normal((rows, cols))).astype(np.float32)


def bf16(a):
    """round to the nearest bfloat16 (ties to even), kept as float32"""
    u = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def stats_arr(st):
    return np.array([st.total_entries, st.nonzeros_before, st.nonzeros_after, st.dropped], dtype=np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default="", help="regenerate one fixture set (e.g. fp8)")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import srelu24 as R  # the reference package

    OUT.mkdir(parents=True, exist_ok=True)
    if args.only == "fp8":
        make_fp8(R)
        return
    if args.only == "nonfinite":
        make_nonfinite(R)
        return

    # ---------------------------------------------------------------- sparsifiers
    cases = {}
    kats = [np.array([[1, -2, 0, 0.5]], np.float32), np.array([[0, 0, 5, 0]], np.float32),
            np.array([[1, -1, 2, 0]], np.float32), np.zeros((2, 8), np.float32)]
    for i, a in enumerate(kats):
        s, m, st = R.sparsify_token_wise(a)
        cases[f"kat{i}_a"] = a
        cases[f"kat{i}_values"] = s.values
        cases[f"kat{i}_meta"] = s.meta
        cases[f"kat{i}_mask"] = m
        cases[f"kat{i}_stats"] = stats_arr(st)
    for i, (rows, cols, p, seed) in enumerate([(64, 128, 0.3, 1), (32, 256, 0.1, 2), (16, 64, 0.9, 3)]):
        a = bern(rng(seed), rows, cols, p)
        a[0, :4] = [2.0, -2.0, 2.0, 0.0]  # three-way magnitude tie
        s, m, st = R.sparsify_token_wise(a)
        cases[f"tok{i}_a"] = a
        cases[f"tok{i}_values"] = s.values
        cases[f"tok{i}_meta"] = s.meta
        cases[f"tok{i}_mask"] = m
        cases[f"tok{i}_stats"] = stats_arr(st)
        f, fm, fst = R.sparsify_feature_wise(a)
        cases[f"feat{i}_values"] = f.values
        cases[f"feat{i}_meta"] = f.meta
        cases[f"feat{i}_mask"] = fm
        cases[f"feat{i}_stats"] = stats_arr(fst)
        kept = R.decompress(s)
        c = R.compress_token_wise_with_mask(kept, m)
        cases[f"cmp{i}_values"] = c.values
        cases[f"cmp{i}_meta"] = c.meta
        b = rng(seed + 50).standard_normal((cols, 8)).astype(np.float32)
        cases[f"spg{i}_b"] = b
        cases[f"spg{i}_out"] = R.sp_gemm(s, b)
        bt = rng(seed + 60).standard_normal((rows, 8)).astype(np.float32)
        cases[f"spgt{i}_b"] = bt
        cases[f"spgt{i}_out"] = R.sp_gemm_t(f, bt)
    np.savez_compressed(OUT / "sparse24.npz", **cases)

    # ---------------------------------------------------------------- plan / permutation / split GEMM
    cases = {}
    plan_cases = [(np.array([0, 5, 1, 9]), 0.5), (np.array([3, 3, 3, 3]), 0.5), (np.zeros(4096, np.int64), 0.95),
                  (np.arange(8), 1.0), (np.arange(8), 0.0), (np.array([5, 1, 5, 1, 0, 7, 7, 2, 2, 2]), 0.29)]
    r = rng(2)
    for _ in range(6):
        h = int(r.integers(1, 300))
        plan_cases.append((r.integers(0, 17, h), float(r.random())))
    for i, (counts, ratio) in enumerate(plan_cases):
        plan = R.partition_features(counts, ratio)
        cases[f"plan{i}_counts"] = np.asarray(counts, np.int64)
        cases[f"plan{i}_ratio"] = np.array([ratio])
        cases[f"plan{i}_sparse"] = plan.sparse_features
        cases[f"plan{i}_dense"] = plan.dense_features
    for i, (seed, n) in enumerate([(0, 16), (3, 100), (0, 4096), (7, 1), (11, 37)]):
        cases[f"perm{i}_seed"] = np.array([seed])
        cases[f"perm{i}_p"] = R.make_permutation(seed, n)
    for i, seed in enumerate(range(5, 9)):
        rr = rng(seed)
        a = bern(rr, 16, 12, 0.3)
        _, mask, _ = R.sparsify_token_wise(a)
        b = rr.standard_normal((16, 6)).astype(np.float32)
        plan = R.partition_features(R.column_nonzero_counts(a), 0.75)
        cases[f"split{i}_a"] = a
        cases[f"split{i}_mask"] = mask
        cases[f"split{i}_b"] = b
        cases[f"split{i}_out"] = R.split_gemm_t(a, mask, b, plan)
        cases[f"split{i}_sparse"] = plan.sparse_features
        cases[f"split{i}_dense"] = plan.dense_features
    np.savez_compressed(OUT / "splitgemm.npz", **cases)

    # ---------------------------------------------------------------- full FFN
    cases = {}
    configs = {
        "recipe": R.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
                              permute_tokens=True),
        "dense": R.FfnConfig(),
        "fwd_sparse": R.FfnConfig(forward_mode="sparse24"),
        "naive_masked": R.FfnConfig(forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True),
        "split_nomask": R.FfnConfig(forward_mode="sparse24", backward_mode="split_masked"),
        "recipe_seed3_r05": R.FfnConfig(forward_mode="sparse24", backward_mode="split_masked",
                                        mask_grad_with_fwd=True, permute_tokens=True, permute_seed=3,
                                        split_ratio=0.5),
    }
    for shape_i, (n, d, h) in enumerate([(32, 8, 16), (128, 32, 64)]):
        rr = rng(100 + shape_i)
        x = rr.standard_normal((n, d)).astype(np.float32)
        w1 = (rr.standard_normal((d, h)) / np.sqrt(d)).astype(np.float32)
        w2 = (rr.standard_normal((h, d)) / np.sqrt(h)).astype(np.float32)
        g = rr.standard_normal((n, d)).astype(np.float32)
        p = R.FfnParams(w1=w1, w2=w2)
        tag = f"s{shape_i}"
        cases[f"{tag}_x"], cases[f"{tag}_w1"], cases[f"{tag}_w2"], cases[f"{tag}_g"] = x, w1, w2, g
        for name, cfg in configs.items():
            out, cache = R.ffn_forward(x, p, cfg)
            grads = R.ffn_backward(g, cache, p, cfg)
            k = f"{tag}_{name}"
            cases[f"{k}_out"] = out
            cases[f"{k}_d_w1"] = grads.d_w1
            cases[f"{k}_d_w2"] = grads.d_w2
            cases[f"{k}_d_x"] = grads.d_x
            cases[f"{k}_census"] = np.array([int(e.sparse) for e in cache.census + grads.census])
            if cache.fwd_mask is not None:
                cases[f"{k}_mask"] = cache.fwd_mask
                cases[f"{k}_stats"] = stats_arr(cache.stats)
            if cache.plan is not None:
                cases[f"{k}_plan_sparse"] = cache.plan.sparse_features
    np.savez_compressed(OUT / "ffn.npz", **cases)

    # ---------------------------------------------------------------- file formats (S24C / S24M)
    import tempfile

    cases = {}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        fmt_cases = [("tok", "token", 8, 16, 0.4, 51), ("feat", "feature", 16, 12, 0.4, 52),
                     ("odd", "token", 3, 4, 0.6, 53)]  # 3 groups: padded last metadata byte
        for tag, orient, rows, cols, p, seed in fmt_cases:
            a = bern(rng(seed), rows, cols, p)
            s, _, _ = (R.sparsify_token_wise(a) if orient == "token" else R.sparsify_feature_wise(a))
            R.write_sparse(td / f"{tag}.s24c", s)
            blob = (td / f"{tag}.s24c").read_bytes()
            back = R.read_sparse(td / f"{tag}.s24c")
            assert np.array_equal(back.values, s.values) and np.array_equal(back.meta, s.meta)
            cases[f"{tag}_a"] = a
            cases[f"{tag}_values"] = s.values
            cases[f"{tag}_meta"] = s.meta
            cases[f"{tag}_bytes"] = np.frombuffer(blob, dtype=np.uint8)
        m = rng(54).standard_normal((5, 7)).astype(np.float32)
        R.write_matrix(td / "m.s24m", m)
        cases["mat_a"] = m
        cases["mat_bytes"] = np.frombuffer((td / "m.s24m").read_bytes(), dtype=np.uint8)
        # malformed files and the reference's error (message with byte offset)
        good = (td / "tok.s24c").read_bytes()
        bad = {"magic": b"XXXX" + good[4:], "short": good[:10], "trunc": good[:-1],
               "version": good[:4] + (2).to_bytes(4, "little") + good[8:],
               "orient": good[:8] + bytes([7]) + good[9:]}
        mgood = (td / "m.s24m").read_bytes()
        bad.update({"m_magic": b"ABCD" + mgood[4:], "m_trunc": mgood[:-3], "m_trail": mgood + b"\0\0\0\0",
                    "m_nan": mgood[:16] + np.float32(np.nan).tobytes() + mgood[20:]})
        for k, blob in bad.items():
            (td / "bad").write_bytes(blob)
            try:
                (R.read_matrix if k.startswith("m_") else R.read_sparse)(td / "bad")
                err = ""
            except R.FormatError as e:
                err = str(e)
            cases[f"bad_{k}_bytes"] = np.frombuffer(blob, dtype=np.uint8)
            cases[f"bad_{k}_error"] = np.array(err)
    np.savez_compressed(OUT / "formats.npz", **cases)
    make_nonfinite(R)
    for f in sorted(OUT.glob("*.npz")):
        print(f, f.stat().st_size)


def make_nonfinite(R):
    """NaN / Inf through the reference (it accepts them: ffn_forward and the
    sparsifiers check shape and dtype, not finiteness): numpy's maximum keeps
    NaN, count_nonzero counts it, the stable argsort ranks it below zero.
    Also the masked feature-wise sparsifier (sparse24.py:118-129) on random
    masks, including the reference's all-ones / all-zeros KATs
    (tests/test_sparse24.py:119-140)."""
    cases = {}
    r = rng(300)
    for i, (rows, cols) in enumerate([(16, 32), (64, 64)]):
        a = bern(r, rows, cols, 0.5)
        a[r.random((rows, cols)) < 0.08] = np.nan
        a[r.random((rows, cols)) < 0.03] = np.inf
        a[r.random((rows, cols)) < 0.03] = -np.inf
        a[0, :4] = [np.nan, 0.0, 0.0, 0.0]      # NaN ranks below zeros
        a[0, 4:8] = [np.nan, np.nan, 1.0, np.nan]  # NaN kept only with < 2 others above it
        a[1, :4] = [np.nan, np.nan, np.nan, np.nan]
        s, m, st = R.sparsify_token_wise(a)
        cases[f"tok{i}_a"] = a
        cases[f"tok{i}_values"] = s.values
        cases[f"tok{i}_meta"] = s.meta
        cases[f"tok{i}_mask"] = m
        cases[f"tok{i}_stats"] = stats_arr(st)
        f, fm, fst = R.sparsify_feature_wise(a)
        cases[f"feat{i}_values"] = f.values
        cases[f"feat{i}_meta"] = f.meta
        cases[f"feat{i}_stats"] = stats_arr(fst)
        cases[f"counts{i}"] = R.column_nonzero_counts(a)
        cases[f"plan{i}_sparse"] = R.partition_features(R.column_nonzero_counts(a), 0.75).sparse_features
    # full FFN, recipe, with NaN / Inf in a few W1 columns (mixed groups) and
    # one NaN input row
    # (bf16-representable inputs: the device path computes on bf16 operands)
    n, d, h = 32, 8, 16
    rr = rng(301)
    x = bf16(rr.standard_normal((n, d)))
    w1 = bf16(rr.standard_normal((d, h)) / np.sqrt(d))
    w2 = bf16(rr.standard_normal((h, d)) / np.sqrt(h))
    g = bf16(rr.standard_normal((n, d)))
    w1[:, 2] = np.nan
    w1[0, 5] = np.inf
    w1[3, 9] = np.nan
    x[7, 3] = np.nan
    cfg = R.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True,
                      permute_tokens=True)
    out, cache = R.ffn_forward(x, R.FfnParams(w1=w1, w2=w2), cfg)
    grads = R.ffn_backward(g, cache, R.FfnParams(w1=w1, w2=w2), cfg)
    cases.update(ffn_x=x, ffn_w1=w1, ffn_w2=w2, ffn_g=g, ffn_out=out, ffn_pre=cache.pre_act,
                 ffn_mask=cache.fwd_mask, ffn_stats=stats_arr(cache.stats),
                 ffn_plan_sparse=cache.plan.sparse_features, ffn_d_x=grads.d_x, ffn_d_w1=grads.d_w1,
                 ffn_d_w2=grads.d_w2)
    # masked feature-wise
    a = rng(4).standard_normal((8, 8)).astype(np.float32)
    for tag, mask in (("ones", np.ones((8, 8), bool)), ("zeros", np.zeros((8, 8), bool))):
        sm, mm, st = R.sparsify_feature_wise_masked(a, mask)
        cases[f"masked_{tag}_a"], cases[f"masked_{tag}_mask"] = a, mask
        cases[f"masked_{tag}_values"], cases[f"masked_{tag}_meta"] = sm.values, sm.meta
        cases[f"masked_{tag}_stats"] = stats_arr(st)
    rm = rng(6)
    for i in range(4):
        a = rm.standard_normal((8 * (i + 1), 12)).astype(np.float32)
        mask = rm.random(a.shape) < 0.5
        sm, mm, st = R.sparsify_feature_wise_masked(a, mask)
        cases[f"masked_r{i}_a"], cases[f"masked_r{i}_mask"] = a, mask
        cases[f"masked_r{i}_values"], cases[f"masked_r{i}_meta"] = sm.values, sm.meta
        cases[f"masked_r{i}_keep"] = mm
        cases[f"masked_r{i}_stats"] = stats_arr(st)
    with np.errstate(all="ignore"):
        np.savez_compressed(OUT / "nonfinite.npz", **cases)


def make_fp8(R):
    """e4m3 encode / quantize / GEMM known answers and the fp8 FFN configs
    (ref matcore.py:113-261, ffn.py:206-268)."""
    from srelu24 import matcore as RM

    cases = {}
    dec = RM._E4M3_DECODE
    finite = dec[~np.isnan(dec)]
    pos = np.unique(np.abs(finite))
    mids = (pos[1:] + pos[:-1]) / 2
    r = rng(300)
    xs = np.concatenate([finite, mids, -mids, pos * 1.0001, pos * 0.9999, [1e9, -1e9, 449.0, 464.0, 480.0, 2.0**-10,
                         -2.0**-10, 2.0**-11, 3 * 2.0**-11, -0.0, 0.0]],
                        ).astype(np.float64)
    xs = np.concatenate([xs, r.standard_normal(4096) * 10.0 ** r.uniform(-4, 3, 4096)])
    cases["enc_x"] = xs
    cases["enc_codes"] = RM.e4m3_encode(xs)
    cases["dec_table"] = dec
    for i, (rows, cols, seed, zero_row) in enumerate([(16, 32, 301, True), (8, 64, 302, False), (33, 40, 303, True)]):
        a = rng(seed).standard_normal((rows, cols)).astype(np.float32) * np.float32(10.0 ** (i - 1))
        if zero_row:
            a[1] = 0.0
            a[:, 2] = 0.0
        for axis in ("rows", "cols"):
            q = R.fp8_quantize_rowwise(a, axis)
            cases[f"q{i}_{axis}_codes"] = q.codes
            cases[f"q{i}_{axis}_scales"] = q.scales
        cases[f"q{i}_a"] = a
    a = rng(109).uniform(-1, 1, (32, 48)).astype(np.float32)
    b = rng(110).uniform(-1, 1, (48, 24)).astype(np.float32)
    cases["gemm_a"], cases["gemm_b"] = a, b
    cases["gemm_out"] = R.fp8_gemm_rowwise(R.fp8_quantize_rowwise(a, "rows"), R.fp8_quantize_rowwise(b, "cols"))
    recipe = dict(forward_mode="sparse24", backward_mode="split_masked", mask_grad_with_fwd=True, permute_tokens=True)
    configs = {
        "recipe_f8fwd": R.FfnConfig(**recipe, fp8_emulation=True),
        "recipe_f8all": R.FfnConfig(**recipe, fp8_emulation=True, fp8_backward=True),
        "dense_f8all": R.FfnConfig(fp8_emulation=True, fp8_backward=True),
        "naive_f8all": R.FfnConfig(forward_mode="sparse24", backward_mode="naive_sparse", mask_grad_with_fwd=True,
                                   fp8_emulation=True, fp8_backward=True),
        "split_nomask_f8all": R.FfnConfig(forward_mode="sparse24", backward_mode="split_masked", fp8_emulation=True,
                                          fp8_backward=True),
    }
    for shape_i, (n, d, h) in enumerate([(32, 8, 16), (64, 32, 64)]):
        rr = rng(400 + shape_i)
        x = rr.standard_normal((n, d)).astype(np.float32)
        w1 = (rr.standard_normal((d, h)) / np.sqrt(d)).astype(np.float32)
        w2 = (rr.standard_normal((h, d)) / np.sqrt(h)).astype(np.float32)
        g = rr.standard_normal((n, d)).astype(np.float32)
        p = R.FfnParams(w1=w1, w2=w2)
        tag = f"s{shape_i}"
        cases[f"{tag}_x"], cases[f"{tag}_w1"], cases[f"{tag}_w2"], cases[f"{tag}_g"] = x, w1, w2, g
        for name, cfg in configs.items():
            out, cache = R.ffn_forward(x, p, cfg)
            grads = R.ffn_backward(g, cache, p, cfg)
            k = f"{tag}_{name}"
            cases[f"{k}_out"] = out
            cases[f"{k}_d_w1"] = grads.d_w1
            cases[f"{k}_d_w2"] = grads.d_w2
            cases[f"{k}_d_x"] = grads.d_x
            if cache.act_sparse is not None:
                cases[f"{k}_act_values"] = cache.act_sparse.values
    # the reference's known answer: selection sees the unquantized values
    # (ref tests/test_ffn.py:360-367)
    p = R.FfnParams(w1=np.eye(4, dtype=np.float32), w2=np.eye(4, dtype=np.float32))
    x = np.array([[3.01, 3.0, 2.99, -1.0]] * 4, np.float32)
    _, cache = R.ffn_forward(x, p, R.FfnConfig(forward_mode="sparse24", fp8_emulation=True))
    cases["kat_sel_x"] = x
    cases["kat_sel_meta"] = cache.act_sparse.meta
    np.savez_compressed(OUT / "fp8.npz", **cases)
    print(OUT / "fp8.npz", (OUT / "fp8.npz").stat().st_size)


if __name__ == "__main__":
    main()
