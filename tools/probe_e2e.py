"""e2e (staged) step of the bench: per-call times and one CUDA timeline (C3 workload)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1512_06235_b200.bank import HostBank
from paper_1512_06235_b200.guided import HostPairs, match_pairs_rows_staged

dev = torch.device("cuda", 0)
scene, wl, ok, snap = bench.build_workload(320, with_snapshot=True)
ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
host = HostBank(scene.feature_sets)
pinned = torch.empty((int(sum(len(x) for x in ql)), 4), dtype=torch.int32, pin_memory=True)
args = (wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
hp = HostPairs(host, *args)
sb = [None]
def step(**kw):
    rows, sb[0] = match_pairs_rows_staged(host, *args, device=dev, pinned=pinned, bank=sb[0], host_pairs=hp, **kw)
    return rows
for kw in ({}, {"chunk_pairs": 2048}, {"chunk_pairs": 2700}, {"first_chunk_pairs": 256}):
    for _ in range(2): step(**kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); step(**kw); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(kw, f"median {np.median(ts):.2f} ms  all " + " ".join(f"{t:.1f}" for t in ts), flush=True)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step(); torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
