"""Aggregate an ncu source page (cuda,sass) by CUDA source line: executed
warp instructions and stall samples.  usage: ncu_lines.py report.ncu-rep [kernel-regex]"""
import csv, io, subprocess, sys, re
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; cur = None; agg = {}
for r in rows:
    if r and r[0] == "Address" or (len(r) > 2 and r[1] == "Source" and r[0] in ("Line No", "Address")):
        hdr = r; continue
    if hdr is None or len(r) < 6: continue
    d = dict(zip(hdr, r))
    if r[0] and r[0].isdigit():
        cur = (int(r[0]), r[1][:90]); continue
    if cur is None: continue
    try:
        ex = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += ex; a[1] += smp
tot_i = sum(v[0] for v in agg.values()) or 1; tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {tot_i}, stall samples {tot_s}")
KEY = 0 if "--by-instr" in sys.argv else 1
for (ln, src), (i, s) in sorted(agg.items(), key=lambda x: -x[1][KEY])[:45]:
    print(f"{ln:5d} instr {i/tot_i*100:5.1f}%  stall {s/tot_s*100:5.1f}%  {src}")
