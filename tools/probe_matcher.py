"""Quick matcher timing probe (not the bench): C3 recipe at N cameras."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs, prepare_pairs

ncam = int(sys.argv[1]) if len(sys.argv) > 1 else 64
t0 = time.time()
scene, snap = scenes.build("C3", n_cameras=ncam)
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
print(f"setup {time.time()-t0:.1f}s  cams={ncam} pairs={len(ok)} mean_q={np.mean([len(x) for x in ql]):.0f}", flush=True)
bank = FeatureBank(scene.feature_sets)
inp = prepare_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
bank.grid(10.0)
for chunk in (64, 256, 1024):
    for it in range(4):
        torch.cuda.synchronize(); s = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, device_inputs=inp, chunk_pairs=chunk)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    n = int(res.count.sum())
    print(f"chunk={chunk}: {ms:.2f} ms  -> {len(ok)/ms*1e3:.0f} pairs/s  {ms*1e3/len(ok):.2f} us/pair  matches={n}", flush=True)
