"""One resident C3 matcher step (the bench's device step) after two warm-up steps,
for an ncu launch list of that step alone:
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(?!at::)' -s 8 --csv \
      --log-file out.csv python tools/one_step.py
(4 library launches per step: plan, setup, match, compact; -s 8 skips the warm-ups)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs, prepare_pairs

scene, snap = scenes.build("C3", n_cameras=320)
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
bank = FeatureBank(scene.feature_sets)
inp = prepare_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
bank.grid(10.0)
torch.cuda.synchronize()
for _ in range(3):
    res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, device_inputs=inp)
torch.cuda.synchronize()
print("matches", int(res.count.sum()))
