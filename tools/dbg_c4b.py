"""Debug: the C4 bench-parity sample (500 cameras, 64 pairs) with per-kernel sync checks."""
import os, sys
os.environ["MSFM_SYNC_CHECK"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs
scene, snap = scenes.build("C4")
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
pick = np.sort(np.random.default_rng(1).choice(ok, size=64, replace=False))
ql = [wl.untracked[int(wl.q_img[k])] for k in pick]
print("nq", sorted(len(x) for x in ql)[:5], max(len(x) for x in ql), flush=True)
bank = FeatureBank(scene.feature_sets)
for sub in (pick[:8], pick[:32], pick):
    qq = [wl.untracked[int(wl.q_img[k])] for k in sub]
    try:
        res = match_pairs(bank, wl.q_img[sub], wl.t_img[sub], wl.F[sub], qq)
        torch.cuda.synchronize()
        print(len(sub), "ok", int(res.count.sum()), flush=True)
    except Exception as e:
        print(len(sub), "FAIL", e, flush=True)
        break
