"""Coarse match-graph probe: C2 scene (100 cameras, 8k features), eta = 20 tiers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import _lib, scenes
from paper_1512_06235_b200.coarse import build_coarse_matchgraph

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
scene, snap = scenes.build("C2", n_cameras=n)
store = scene.store()
store.apply_eta(20.0)
print("tiers", int(np.mean([fs.coarse_count for fs in store.sets.values()])))
g = build_coarse_matchgraph(store.sets, on_overflow="drop")
torch.cuda.synchronize()
_lib.profile_enable(True)
t0 = time.perf_counter()
g = build_coarse_matchgraph(store.sets, on_overflow="drop")
torch.cuda.synchronize()
dt = time.perf_counter() - t0
names = ("knn_tc_kernel", "f_hyp_kernel", "f_score_kernel", "f_refit_kernel")
k = {nm: _lib.profile_read(nm) for nm in names}
_lib.profile_enable(False)
P = n * (n - 1) // 2
print(f"cams={n} pairs={P} edges={len(g.edges)} overflow={len(g.overflow_pairs)} wall {dt*1e3:.1f} ms ({P/dt:.0f} pairs/s)  " +
      "  ".join(f"{nm} {v[0]:.2f}ms/{v[1]}" for nm, v in k.items()))

import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
build_coarse_matchgraph(store.sets, on_overflow="drop")
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    build_coarse_matchgraph(store.sets, on_overflow="drop")
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/coarse_trace.json")
