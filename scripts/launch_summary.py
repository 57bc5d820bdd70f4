"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`):
the kernels of the last recipe step in launch order with their durations, and
per-kernel totals. Durations are ncu's serialised, cold-cache launches: use
the SHARES, not the absolute sum, against bench.py's step time.

usage: python scripts/launch_summary.py launches.csv [--step-marker EpiFwd1]
"""

import argparse
import csv
import re


def short(name: str) -> str:
    m = re.match(r"void s24::gemm_kernel<s24::GemmCfg<(\d), (\d), (\d), (\d+), (\d+), (\d), (\d+), (\d)>, s24::(\w+)(<[^>]*>)?", name)
    if m:
        sp, amn, bmn, bn, st, cg, ew, mc, epi, tp = m.groups()
        kind = "spmm 2:4" if sp == "1" else "gemm"
        return f"{kind} [{epi}{tp or ''}] A{'MN' if amn == '1' else 'K'} B{'MN' if bmn == '1' else 'K'} BN{bn} st{st}"
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "")[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--step-marker", default="EpiFwd1", help="kernel that starts a recipe step (K1)")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    ks = [(int(r[ii]), r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if r[vi]]
    starts = [j for j, (_, k, _) in enumerate(ks) if args.step_marker in k]
    # the last complete step: from the second-to-last K1 (minus its gather) to the last K1
    a, b = starts[-2], starts[-1]
    while a > 0 and "gather" in ks[a - 1][1]:
        a -= 1
    while b > 0 and "gather" in ks[b - 1][1]:
        b -= 1
    step = [k for k in ks[a:b] if "FillFunctor" not in k[1]]
    tot = sum(v for _, _, v in step)
    print(f"# one recipe step, {len(step)} kernels, serialised sum {tot / 1e3:.1f} us (ncu, cold cache)")
    print(f"{'id':>5}  {'us':>8}  {'share':>6}  kernel")
    for i, k, v in step:
        print(f"{i:5d}  {v / 1e3:8.1f}  {v / tot:6.1%}  {short(k)}")


if __name__ == "__main__":
    main()
