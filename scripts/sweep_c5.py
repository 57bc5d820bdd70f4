"""c5 (BASELINE configs[4]): activation-sparsity sweep at the
7B-class shape.

For each target sparsity s: the recipe fwd+bwd step (graph) vs the dense twin
(timed by bench.py in interleaved blocks, so both see the same clocks), the
drop fractions (token-wise forward, feature-wise backward for act and g_pre),
the sparse TFLOPS, and the tensor-pipe utilisation of every GEMM of the step
(achieved dense-equivalent TFLOP/s over the measured peak: 2:4 GEMMs against
twice the dense bf16 peak, from bench.py's per-kernel CUDA-event pass). A
point whose two arms ran at median SM clocks more than 5% apart is flagged
"rejected" (its speedup is a clock artefact) and re-run once. One bench.py
process per point (c4 shape: 32768 tokens, d=4096, h=16384).

usage: python scripts/sweep_c5.py [--out profiles/r02/sweep_c5.json] [--config c4]
"""

import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LEVELS = [0.5, 0.6, 0.7, 0.8, 0.85, 0.9, 0.95, 0.98]
IID_DROP = {0.5: 0.1875, 0.6: 0.128, 0.7: 0.0765, 0.8: 0.036, 0.85: 0.0208, 0.9: 0.0095, 0.95: 0.00244,
            0.98: 0.0004}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02" / "sweep_c5.json"))
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    rows = []
    for s in LEVELS:
        for attempt in range(2):
            cmd = [sys.executable, str(ROOT / "bench.py"), "--config", args.config, "--sparsity", str(s), "--steps",
                   str(args.steps), "--warmup", "3", "--no-e2e", "--no-cpu"]
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except (IndexError, ValueError):
                print(f"s={s}: failed\n{r.stderr[-2000:]}", file=sys.stderr)
                d = None
                break
            mhz, dmhz = d["clocks"].get("sm_mhz") or 0, (d["dense_twin"].get("clocks") or {}).get("sm_mhz") or 0
            rejected = not (mhz and dmhz) or abs(mhz - dmhz) > 0.05 * max(mhz, dmhz)
            if not rejected:
                break
        if d is None:
            continue
        tensor = {k["kernel"]: round(k["frac"], 3) for k in d["kernels"] if k["unit"] == "TFLOP/s"}
        row = {"sparsity": s, "ms_per_step": d["ms_per_step"], "dense_ms_per_step": d["dense_twin"]["ms_per_step"],
               "speedup_vs_dense": d["speedup_vs_dense"], "sparse_tflops": d["sparse_tflops"],
               "iid_token_wise_drop": IID_DROP[s], **d["drops"], "clocks": d["clocks"],
               "dense_clocks": d["dense_twin"].get("clocks"), "clock_mismatch_rejected": rejected,
               "tensor_pipe_frac_per_gemm": tensor,
               "fp8_ms_per_step": (d.get("fp8_variant") or {}).get("ms_per_step"),
               "fp8_speedup_vs_dense_bf16": (d.get("fp8_variant") or {}).get("speedup_vs_dense_bf16"),
               "fp8_speedup_vs_dense_fp8": (d.get("fp8_variant") or {}).get("speedup_vs_dense_fp8")}
        rows.append(row)
        print(json.dumps(row), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(rows, indent=1))
    print(f"\n{'s':>5} {'ms':>7} {'dense':>7} {'speedup':>8} {'TF/s':>7} {'fwd drop':>9} {'iid':>7} "
          f"{'act fw':>7} {'g fw':>7} {'fp8 ms':>7} {'MHz':>6}")
    for r in rows:
        print(f"{r['sparsity']:5.2f} {r['ms_per_step']:7.3f} {r['dense_ms_per_step']:7.3f} {r['speedup_vs_dense']:8.3f} "
              f"{r['sparse_tflops']:7.0f} {r['fwd_token_wise_dropped_fraction']:9.4%} {r['iid_token_wise_drop']:7.3%} "
              f"{r['bwd_act_feature_wise_dropped_fraction']:7.3%} {r['bwd_grad_feature_wise_dropped_fraction']:7.3%} "
              f"{r['fp8_ms_per_step'] or 0:7.3f} {r['clocks'].get('sm_mhz') or 0:6.0f}")


if __name__ == "__main__":
    main()
