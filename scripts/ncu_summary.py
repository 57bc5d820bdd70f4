"""Summarise an ncu report: headline metrics + per-opcode instruction mix and
stall samples from the SASS source page. usage: ncu_summary.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "gpc__cycles_elapsed.max.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg"]
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            print(f"{h:70s} {vals[i][:100]} {units[i]}")
            break
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h2 = srows[1]
ie, sc, st = h2.index("Instructions Executed"), h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)")
byop, stall, tot = collections.Counter(), collections.Counter(), 0
for r in srows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    toks = r[sc].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    byop[op] += n
    stall[op] += int(r[st] or 0)
    tot += n
print("total warp instructions", tot)
for op, n in byop.most_common(14):
    print(f"  {op:10s} {n:12d} {100*n/tot:5.1f}%  stall-samples {stall[op]}")
print("top stall ops:", stall.most_common(8))
