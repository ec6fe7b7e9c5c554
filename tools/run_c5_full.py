"""All of BASELINE configs[4]'s densify matching and its track merge on ONE B200:
the C5 scene (3000 cameras, 16k features/img, all registered, ~467k covisible
pairs), matched in waves of pairs with each wave's matches kept on the device as
(u, v, dist) over bank rows, then one device track merge of every match — the
computation rank 0 performs after the NVLink gather of the other ranks' matches
in an 8-GPU run.  Host synthesis is reported, not counted.

    python tools/run_c5_full.py [wave_pairs=60000] [n_cameras=3000]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank, HostBank
from paper_1512_06235_b200.densify import merge_tracks_nodes
from paper_1512_06235_b200.guided import match_pairs, prepare_pairs

wave = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
n_cam = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
t0 = time.perf_counter()
scene = scenes.generate_scene(scenes.spec_for("C5", n_cam))
snap = scenes.coarse_snapshot(scene, list(range(n_cam)))
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
print(f"C5: {n_cam} cameras, {len(ok)} pairs (host synthesis {time.perf_counter() - t0:.0f} s)",
      flush=True)
host = HostBank(scene.feature_sets)
bank = FeatureBank(host=host)
bank.grid(10.0)
torch.cuda.synchronize()
dev = bank.device
parts = []
n_match = 0
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
# each wave's pair tables built and uploaded before the timed loop (as the bench's
# resident step does); the loop below is device matching + packing only
waves = []
t_prep = time.perf_counter()
for w0 in range(0, len(ok), wave):
    sel = ok[w0:w0 + wave]
    ql = [wl.untracked[int(wl.q_img[k])] for k in sel]
    waves.append((sel, ql, prepare_pairs(bank, wl.q_img[sel], wl.t_img[sel], wl.F[sel], ql)))
torch.cuda.synchronize()
print(f"  pair tables of {len(waves)} waves prepared on the host and uploaded in "
      f"{(time.perf_counter() - t_prep) * 1e3:.0f} ms (outside the timed matching)", flush=True)
e0.record()
for sel, ql, inp in waves:
    res = match_pairs(bank, wl.q_img[sel], wl.t_img[sel], wl.F[sel], ql, device_inputs=inp)
    rows, n = res.packed()
    del res
    qoff = torch.from_numpy(bank.offsets[bank.slots(wl.q_img[sel])]).to(dev)
    toff = torch.from_numpy(bank.offsets[bank.slots(wl.t_img[sel])]).to(dev)
    pk = rows[:, 0].long()
    parts.append(((qoff[pk] + (rows[:, 1] & 0xFFFF).long()).to(torch.int32),
                  (toff[pk] + ((rows[:, 1] >> 16) & 0xFFFF).long()).to(torch.int32),
                  rows[:, 2].contiguous().view(torch.float32).clone()))
    del rows, pk
    n_match += int(n)
e1.record()
torch.cuda.synchronize()
ms_match = e0.elapsed_time(e1)
print(f"  matching: {len(ok)} pairs in {ms_match:.0f} ms ({len(ok) / ms_match * 1e3:.0f} pairs/s), "
      f"{n_match} matches; device memory in use {torch.cuda.memory_allocated() / 1e9:.1f} GB",
      flush=True)
u = torch.cat([p[0] for p in parts])
v = torch.cat([p[1] for p in parts])
dist = torch.cat([p[2] for p in parts])
del parts
torch.cuda.empty_cache()
slot = bank.slots(snap.track_img)
tnode = (bank.offsets[slot] + snap.track_fid).astype(np.int32)
torch.cuda.synchronize()
e0.record()
nodes, owners, offs = merge_tracks_nodes(bank, u, v, dist, snap.track_ptr, tnode)
e1.record()
torch.cuda.synchronize()
ms_merge = e0.elapsed_time(e1)
print(f"  track merge: {len(u)} edges over {bank.n_total} bank rows -> {len(owners)} tracks "
      f"({int((np.asarray(owners) < 0).sum())} new, {len(nodes)} fresh nodes) in {ms_merge:.0f} ms "
      f"({len(u) / ms_merge / 1e6:.2f} G edges/s)", flush=True)
print(f"  device memory peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
