"""Matcher timing probe (not the bench): C3 recipe at N cameras; reports the
step time and the library's per-kernel CUDA-event times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import _lib, scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs, prepare_pairs

ncam = int(sys.argv[1]) if len(sys.argv) > 1 else 128
chunks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256]
t0 = time.time()
scene, snap = scenes.build("C3", n_cameras=ncam)
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
print(f"setup {time.time()-t0:.1f}s  cams={ncam} pairs={len(ok)}", flush=True)
bank = FeatureBank(scene.feature_sets)
inp = prepare_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
bank.grid(10.0)
for chunk in chunks:
    for it in range(3):
        res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, device_inputs=inp, chunk_pairs=chunk)
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, device_inputs=inp, chunk_pairs=chunk)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    km, kn = _lib.profile_read("match_kernel")
    others = {k: _lib.profile_read(k)[0] for k in ("setup_kernel", "gather_kernel", "compact_kernel")}
    _lib.profile_enable(False)
    n = int(res.count.sum())
    print(f"chunk={chunk}: step {ms:.2f} ms ({ms*1e3/len(ok):.2f} us/pair, {len(ok)/ms*1e3:.0f} pairs/s) "
          f"match_kernel {km:.2f} ms in {kn} launches ({km*1e3/len(ok):.2f} us/pair)  matches={n}", flush=True)
    print("   " + "  ".join(f"{k.replace('_kernel', '')} {v:.3f}" for k, v in others.items()), flush=True)

# workload counters
lib = _lib.load()
cnt = np.zeros(16, np.int64)
lib.msfm_debug_counters(1, None)
res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, device_inputs=inp, chunk_pairs=chunks[-1])
torch.cuda.synchronize()
lib.msfm_debug_counters(1, cnt.ctypes.data)
lib.msfm_debug_counters(0, None)
names = ["supergroups", "members", "gathered", "passing", "sure", "strip rows (clk: SG setup)", "match: tiles clk",
         "(cbstats) annulus member loops | gather clk", "groups", "(cbstats) C' band-edge exact | C' clk", "(cbstats) (cand, group) tests | ratio clk", "setup: lines clk", "setup: groups clk", "setup: scatter+geo clk",
         "setup: chain+shape clk", "setup: members+strips clk"]
P = len(ok)
for k, nme in enumerate(names):
    print(f"  {nme:14s} {cnt[k]:>12d}  per pair {cnt[k]/P:10.1f}  per SG {cnt[k]/max(cnt[0],1):8.2f}")
