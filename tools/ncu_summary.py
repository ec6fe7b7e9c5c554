"""Summarise an ncu report (raw page) and an ncu launch-list CSV into
profiles/*.json / *.txt.  usage:
  ncu_summary.py report.ncu-rep out.json [pairs_per_launch]
  ncu_summary.py --launches launches.csv out.txt"""
import csv, collections, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__cycles_elapsed.avg",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1}

if sys.argv[1] == "--launches":
    rows = list(csv.reader(open(sys.argv[2])))
    hdr = None; agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r: hdr = r; continue
        if hdr is None or len(r) != len(hdr): continue
        d = dict(zip(hdr, r))
        n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("msfm::<unnamed>::", "")
        agg[n][0] += 1; agg[n][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(sys.argv[3], "w") as f:
        f.write("share   launches  avg_us  kernel  (ncu gpu__time_duration.sum, --clock-control none, serialised)\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{v[1]/tot*100:5.1f}%  {v[0]:6d}  {v[1]/v[0]/1e3:9.1f}  {k}\n")
    print(open(sys.argv[3]).read())
    sys.exit(0)

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units, vals = r[0], r[1], r[2]
res = {"report": sys.argv[1].split("/")[-1], "kernel": dict(zip(h, vals)).get("Kernel Name", "")[:120]}
for k in KEYS:
    if k in h:
        i = h.index(k)
        v = float(vals[i].replace(",", "")) if vals[i] not in ("", "n/a") else None
        u = units[i]
        if v is not None and u in SCALE:
            v *= SCALE[u]; u = "byte" if "byte" in u else "s"
        res[k] = {"value": v, "unit": u}
if len(sys.argv) > 3:
    n = float(sys.argv[3])
    dr = res["dram__bytes_read.sum"]["value"] + res["dram__bytes_write.sum"]["value"]
    res["pairs_per_launch"] = n
    res["dram_bytes_per_pair"] = dr / n
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps(res, indent=1))
