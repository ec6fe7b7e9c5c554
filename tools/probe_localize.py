"""Localization-step probe (not the bench): the bench's C2 step (device-flat
correspondences + pnp_batch_flat), wall-clock split + cProfile + CUDA timeline."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank, HostBank
from paper_1512_06235_b200.localize import PointSet, direct_search, gather_pnp_inputs, upload_points
from paper_1512_06235_b200.pnp import pnp_batch_flat

scene, snap, queries = bench.build_localization()
S, n = scenes.track_sums(scene, snap)
pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
host = HostBank({q: scene.feature_sets[q] for q in queries})
Ks = [scene.cameras[q].K for q in queries]
dev = torch.device("cuda")
bank = FeatureBank(host=host, device=dev)
dp = upload_points(pts, dev)
d_xyz = torch.from_numpy(snap.point_xyz).to(dev)
T = {}
PT = {}


def tick(name, t0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    T.setdefault(name, []).append((t - t0) * 1e3)
    return t


def step():
    t0 = time.perf_counter()
    corr = direct_search(bank, pts, queries, device_points=dp, to_host=False)
    t0 = tick("direct_search (kNN + ratio + dedupe)", t0)
    X, uv, toff, todo = gather_pnp_inputs(bank, corr, queries, d_xyz)
    t0 = tick("gather", t0)
    res = pnp_batch_flat(X, uv, toff, [Ks[k] for k in todo], [queries[k] for k in todo], device=dev,
                         timing=PT)
    tick("pnp_batch_flat", t0)
    return res


for _ in range(3):
    step()
T.clear()
for _ in range(10):
    step()
for k, v in T.items():
    print(f"{k:52s} {np.median(v):7.2f} ms")
PT.pop("_t", None)
for k, v in PT.items():
    print(f"   pnp {k:46s} {v * 1e3 / 13:7.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("gpurun_out/loc_trace.json")

# ---- e2e variants: bank refilled then stepped vs staged (4 ranges, kNN per range)
from paper_1512_06235_b200.localize import knn2_tracks_staged
pin_xyz = torch.from_numpy(snap.point_xyz).pin_memory()
b2 = FeatureBank(host=host, device=dev, staged=True)


def e2e(staged, groups=4):
    dp2 = upload_points(pts, dev)
    if staged:
        knn = knn2_tracks_staged(b2, pts, queries, dp2, groups)
    else:
        b2.refill()
        knn = None
    corr = direct_search(b2, pts, queries, device_points=dp2, to_host=False, knn=knn)
    X, uv, toff, todo = gather_pnp_inputs(b2, corr, queries, pin_xyz.to(dev, non_blocking=True))
    return pnp_batch_flat(X, uv, toff, [Ks[k] for k in todo], [queries[k] for k in todo], device=dev)


for name, fn in (("e2e refill", lambda: e2e(False)), ("e2e staged 4", lambda: e2e(True, 4)),
                 ("e2e staged 2", lambda: e2e(True, 2)), ("e2e staged 8", lambda: e2e(True, 8))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:20s} {np.median(ts):7.2f} ms", flush=True)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    e2e(True, 4)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/loc_e2e_trace.json")
