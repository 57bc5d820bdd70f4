"""bench.py's output contract on the CPU: the reference arm's JSON line (it
runs the reference's own CPU path, or the oracle port when baseline/_ref is
absent) and the helpers that attach the committed ncu figures to the roofline."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["steps"] == 1 and line["warmup"] == 1 and line["n_gpus"] == 1
    assert line["value"] > 0 and line["unit"] == "tokens/s" and line["higher_is_better"] is True
    assert line["config"]["workload"].startswith("c2")
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_roofline_helpers_read_committed_ncu_figures():
    import bench

    label = "spmm 2:4 M=8601 N=2048 K=16384"
    traffic, src = bench.measured_traffic(label)
    assert traffic and traffic > 0 and "profiles/r" in src
    feed = bench.operand_feed(label, 3e-4)
    assert feed["unit"] == "TB/s" and 0 < feed["frac"] < 2
    assert feed["achieved"] == pytest.approx(feed["bytes_per_launch"] / 3e-4 / 1e12)
    assert bench.operand_feed("no such kernel", 3e-4) is None
    assert bench.measured_traffic("no such kernel") == (None, None)
