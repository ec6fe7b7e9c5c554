"""kNN kernel probe: C2 workload (2958 points x 80 query images of 8k features)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import _lib, scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.localize import PointSet, knn2_tracks, upload_points

scene, snap = scenes.build("C2")
reg = set(int(i) for i in snap.registered)
queries = [i for i in range(len(scene.cameras)) if i not in reg]
S, n = scenes.track_sums(scene, snap)
pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
bank = FeatureBank({q: scene.feature_sets[q] for q in queries})
dp = upload_points(pts, bank.device)
for _ in range(3):
    knn2_tracks(bank, pts, queries, device_points=dp)
torch.cuda.synchronize()
_lib.profile_enable(True)
for _ in range(5):
    knn2_tracks(bank, pts, queries, device_points=dp)
torch.cuda.synchronize()
ms, k = _lib.profile_read("knn_tc_kernel")
_lib.profile_enable(False)
N = sum(len(scene.feature_sets[q]) for q in queries)
ops = 2.0 * 2 * len(S) * N * 128
print(f"knn: M={len(S)} N={N} {ms/k:.3f} ms/launch  {ops/(ms/k/1e3)/1e12:.0f} TOPS (hw, 2 planes)")
