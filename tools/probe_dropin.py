"""Per-call latency of the reference-shaped drop-ins on one C3 pair (8k features):
guided_match_pair, and pnp_ransac / triangulate_track for scale."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.geometry import fundamental_from_poses
from paper_1512_06235_b200.guided import guided_match_pair

scene, snap = scenes.build("C3", n_cameras=12)
wl = scenes.pair_workload(scene, snap)
k = int(np.flatnonzero(wl.valid)[0])
q, t = int(wl.q_img[k]), int(wl.t_img[k])
fq, ft = scene.feature_sets[q], scene.feature_sets[t]
geom = fundamental_from_poses(scene.cameras[q], scene.cameras[t])
qi = wl.untracked[q]


def timed(name, fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:52s} {np.median(ts):8.2f} ms", flush=True)
    return out


m = timed(f"guided_match_pair ({len(qi)} queries x {len(ft)} targets)",
          lambda: guided_match_pair(fq, ft, geom, query_indices=qi))
print(f"  {len(m)} matches")
# the same pair through the batched API (device inputs prepared once)
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs, prepare_pairs
bank = FeatureBank({q: fq, t: ft})
bank.grid(10.0)
inp = prepare_pairs(bank, [q], [t], geom.F[None], [qi])
timed("match_pairs, one pair, device-resident inputs",
      lambda: match_pairs(bank, [q], [t], geom.F[None], [qi], device_inputs=inp).count.cpu())
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    guided_match_pair(fq, ft, geom, query_indices=qi)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
