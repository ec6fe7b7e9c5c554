"""e2e (staged) step jitter: 30 steps, per-step event and host times, torch-profiler
trace of all of them (gpurun_out/e2e_jitter_trace.json)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1512_06235_b200.bank import HostBank
from paper_1512_06235_b200.guided import HostPairs, match_pairs_rows_staged
from paper_1512_06235_b200 import _lib

dev = torch.device("cuda", 0)
scene, wl, ok, snap = bench.build_workload(320, with_snapshot=True)
ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
host = HostBank(scene.feature_sets)
pinned = torch.empty((int(sum(len(x) for x in ql)), 4), dtype=torch.int32, pin_memory=True)
args = (wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
hp = HostPairs(host, *args)
sb = [None]
def step():
    rows, sb[0] = match_pairs_rows_staged(host, *args, device=dev, pinned=pinned, bank=sb[0], host_pairs=hp)
    return rows
for _ in range(3): step()
torch.cuda.synchronize()
lib = _lib.load()
from torch.profiler import ProfilerActivity, profile
ts, hs = [], []
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for i in range(30):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(); rows = step(); e1.record(); torch.cuda.synchronize()
        hs.append(1e3 * (time.perf_counter() - h0)); ts.append(e0.elapsed_time(e1))
print("event ms:", " ".join(f"{t:.1f}" for t in ts))
print("host  ms:", " ".join(f"{t:.1f}" for t in hs))
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/e2e_jitter_trace.json")
