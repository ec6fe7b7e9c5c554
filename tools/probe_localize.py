"""Localization-step probe (not the bench): C2 workload, wall-clock breakdown."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank, HostBank
from paper_1512_06235_b200.localize import PointSet, direct_search, upload_points
from paper_1512_06235_b200.pnp import pnp_batch

scene, snap, queries = bench.build_localization()
S, n = scenes.track_sums(scene, snap)
pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
host = HostBank({q: scene.feature_sets[q] for q in queries})
Ks = [scene.cameras[q].K for q in queries]
dev = torch.device("cuda")
bank = FeatureBank(host=host, device=dev)
dp = upload_points(pts, dev)


def step():
    t0 = time.perf_counter()
    corrs = direct_search(bank, pts, queries, device_points=dp)
    t1 = time.perf_counter()
    todo = [k for k, c in enumerate(corrs) if len(c) > 16]
    X = [snap.point_xyz[corrs[k][:, 0]] for k in todo]
    uv = [scene.feature_sets[queries[k]].xy[corrs[k][:, 1]].astype(np.float64) for k in todo]
    t2 = time.perf_counter()
    res = pnp_batch(X, uv, [Ks[k] for k in todo], [queries[k] for k in todo], device=dev)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3


for _ in range(3):
    step()
ts = np.array([step() for _ in range(5)])
print("direct_search %.2f ms  gather %.2f ms  pnp_batch %.2f ms" % tuple(ts.mean(0)))
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
