"""Actual SM clock while a kernel of the step runs: one-warp probe CTAs on a
second stream busy-wait 20 us and compare %clock64 with %globaltimer while the
kernel under test loops on the main stream. NVML's clock samples (every few
ms, and not per kernel) do not show the clock a tensor-heavy kernel gets
under the power limit.

usage: python scripts/clock_probe.py [k1|k3|fwdout|dx|dw|dense|k4 ...]"""
import runpy
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2503_16672_b200 import _lib  # noqa: E402


def mhz(out, ctas):
    v = out.view(ctas, 2).cpu().tolist()
    return sorted(round(c / t * 1e3) for c, t in v)


def main():
    kinds = sys.argv[1:] or ["k1", "fwdout", "dw", "k4", "dense"]
    sys.argv = [sys.argv[0], kinds[0], "--iters", "1"]
    g = runpy.run_path(str(ROOT / "scripts" / "gemm_probe.py"), run_name="probe_setup")
    ctas = 8
    out = torch.zeros(2 * ctas, dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream()
    _lib.call("s24_clock_probe", out.data_ptr(), ctas, 20000, side.cuda_stream)
    torch.cuda.synchronize()
    print("idle", mhz(out, ctas))
    for which in kinds:
        call = g["calls"][which]
        seen = []
        for rep in range(6):
            for _ in range(30):
                call()
            _lib.call("s24_clock_probe", out.data_ptr(), ctas, 20000, side.cuda_stream)
            for _ in range(10):
                call()
            torch.cuda.synchronize()
            seen.append(mhz(out, ctas)[ctas // 2])
        print(which, "SM MHz (median of 8 probe CTAs, 6 reps):", seen)


if __name__ == "__main__":
    main()
