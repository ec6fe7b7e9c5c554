"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report
(source page with cuda,sass correlation).  usage: ncu_lines2.py report [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
out = []
fname = None
for i, r in enumerate(rows):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if len(r) > 8 and r[0] and r[0].isdigit():
        try:
            ie = float(r[7] or 0)
            st = float(r[4] or 0)
        except ValueError:
            continue
        out.append((ie, st, f"{fname}:{r[0]}", r[1][:90]))
tot = sum(x[0] for x in out) or 1
ts = sum(x[1] for x in out) or 1
print(f"total warp instructions {tot:.0f}")
for ie, st, where, text in sorted(out, key=lambda x: -x[0])[:top]:
    print(f"{100*ie/tot:6.2f}% inst {100*st/ts:6.2f}% stall  {where:22s} {text}")
