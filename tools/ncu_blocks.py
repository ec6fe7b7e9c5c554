"""Summarise an ncu report of one kernel: headline counters, then SASS basic blocks
(runs of equal execution count) with their instruction and stall shares.
usage: ncu_blocks.py report.ncu-rep [min_share]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "lts__t_sectors.sum.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum"]:
    print(f"{k:70s} {d.get(k)}")
for k in sorted(d):
    if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
        if float(d[k] or 0) >= 0.1:
            print(f"{k:70s} {d[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
data = [(r[ix["Address"]], r[ix["Source"]].strip(), float(r[ix["Instructions Executed"]] or 0),
         float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in rows[2:] if len(r) >= len(h)]
tot = sum(x[2] for x in data) or 1
ts = sum(x[3] for x in data) or 1
print(f"{len(data)} SASS instructions; {tot:.0f} warp instructions executed")
blocks, cur = [], [data[0]]
for x in data[1:]:
    if x[2] == cur[-1][2]:
        cur.append(x)
    else:
        blocks.append(cur)
        cur = [x]
blocks.append(cur)
for b in blocks:
    ex = b[0][2] * len(b)
    s = sum(x[3] for x in b)
    if ex / tot > thr or s / ts > 0.01:
        ops = Counter((x[1].split()[1] if x[1].startswith("@") else x[1].split()[0]).split(".")[0] for x in b)
        print("%s n=%3d exec=%9d %5.2f%% inst %5.2f%% stall  %s" % (
            b[0][0][-5:], len(b), b[0][2], 100 * ex / tot, 100 * s / ts,
            " ".join("%s:%d" % kv for kv in ops.most_common(8))))
