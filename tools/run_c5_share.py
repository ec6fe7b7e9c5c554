"""One rank's share of BASELINE configs[4] (C5: 3000 cameras, 16k features/img)
on one B200: the scene's densify pairs (all cameras registered, k = 300
covisible partners each, ~450k pairs), every ``world``-th pair (rank 0 of an
8-GPU run), geometry-aware matching of that share on the device, then the device
track merge of its matches.  Host synthesis is reported but not part of the
device numbers.

    python tools/run_c5_share.py [world=8] [n_cameras=3000]
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

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n_cam = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
t0 = time.perf_counter()
spec = scenes.spec_for("C5", n_cam)
scene = scenes.generate_scene(spec)
snap = scenes.coarse_snapshot(scene, list(range(n_cam)))
wl = scenes.pair_workload(scene, snap)
ok = np.flatnonzero(wl.valid)
mine = ok[0::world]
t_host = time.perf_counter() - t0
nfeat = int(np.mean([len(fs) for fs in scene.feature_sets.values()]))
print(f"C5 share: {n_cam} cameras, {nfeat} features/img, {len(ok)} pairs in the scene, "
      f"rank 0 of {world}: {len(mine)} pairs (host synthesis {t_host:.0f} s)", flush=True)

imgs = sorted(set(wl.q_img[mine].tolist()) | set(wl.t_img[mine].tolist()))
ql = [wl.untracked[int(wl.q_img[k])] for k in mine]
t0 = time.perf_counter()
host = HostBank({i: scene.feature_sets[i] for i in imgs})
bank = FeatureBank(host=host)
bank.grid(10.0)
inp = prepare_pairs(bank, wl.q_img[mine], wl.t_img[mine], wl.F[mine], ql)
torch.cuda.synchronize()
t_stage = time.perf_counter() - t0
nq = int(inp[5][-1])
print(f"  bank: {len(imgs)} images, {bank.n_total} features ({host.nbytes / 1e9:.1f} GB), "
      f"{nq} query slots; staging + H2D + index {t_stage * 1e3:.0f} ms", flush=True)

res = None
ms = []
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    del res
    res = None
    torch.cuda.synchronize()
    e0.record()
    res = match_pairs(bank, wl.q_img[mine], wl.t_img[mine], wl.F[mine], ql, device_inputs=inp)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
n_match = int(res.count.sum().item())
print(f"  matching: {ms[-1]:.0f} ms ({len(mine) / ms[-1] * 1e3:.0f} pairs/s, "
      f"{ms[-1] * 1e3 / len(mine):.1f} us/pair; runs {', '.join(f'{m:.0f}' for m in ms)} ms), "
      f"{n_match} matches ({n_match / len(mine):.0f}/pair)", flush=True)

# device track merge of the share's matches (densify.py:68-158) over bank rows
rows, _ = res.packed()
del res
qoff = torch.from_numpy(bank.offsets[bank.slots(wl.q_img[mine])]).to(bank.device)
toff = torch.from_numpy(bank.offsets[bank.slots(wl.t_img[mine])]).to(bank.device)
pk = rows[:, 0].long()
u = (qoff[pk] + (rows[:, 1] & 0xFFFF).long()).to(torch.int32).contiguous()
v = (toff[pk] + ((rows[:, 1] >> 16) & 0xFFFF).long()).to(torch.int32).contiguous()
dist = rows[:, 2].contiguous().view(torch.float32)
del rows, pk
in_bank = np.isin(snap.track_img, imgs)
slot = np.array([bank.index_of.get(int(i), 0) for i in snap.track_img], np.int64)
tnode = (bank.offsets[slot] + snap.track_fid)[in_bank].astype(np.int32)
tptr = np.zeros(len(snap.point_xyz) + 1, np.int64)
np.cumsum(np.bincount(np.repeat(np.arange(len(snap.point_xyz)), np.diff(snap.track_ptr))[in_bank],
                      minlength=len(snap.point_xyz)), out=tptr[1:])
torch.cuda.synchronize()
mt = []
for it in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nodes, owners, offs = merge_tracks_nodes(bank, u, v, dist, tptr, tnode)
    e1.record()
    torch.cuda.synchronize()
    mt.append(e0.elapsed_time(e1))
print(f"  track merge: {len(u)} edges -> {len(owners)} tracks "
      f"({int((np.asarray(owners) < 0).sum())} new), {mt[-1]:.0f} ms "
      f"({len(u) / mt[-1] / 1e6:.2f} G edges/s)", flush=True)
print(f"  device memory peak {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
