"""The fine stage end to end on the device at a BASELINE config (default C4:
500 cameras, 16k features/img, every 5th camera in the coarse model M0):

  1. 3D-2D localization of the unregistered images (exact kNN + ratio + one
     point per feature, seeded PnP-RANSAC), localize.py:179-281;
  2. the localized cameras join M0 with their PnP inliers as track links;
  3. densification over all registered cameras: covisibility pairs,
     geometry-aware matching, device track merge, batched multi-view
     triangulation of the new and grown tracks (densify.py:168-286).

Arrays throughout (no per-point Python objects); wall-clock per stage with the
device synchronized.  Accuracy: triangulated positions against the scene's
ground truth for the tracks whose features all see one world point.

    python tools/run_fine_stage.py [C4|C5] [n_cameras]
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
from paper_1512_06235_b200.geometry import fundamental_from_poses
from paper_1512_06235_b200.guided import match_pairs
from paper_1512_06235_b200.localize import PointSet, direct_search, upload_points
from paper_1512_06235_b200.pnp import pnp_batch
from paper_1512_06235_b200.triangulation import triangulate_batch
from paper_1512_06235_b200.types import Camera, DegenerateGeometryError

config = sys.argv[1] if len(sys.argv) > 1 else "C4"
n_cam = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else None
T = {}


def tick(name, t0):
    torch.cuda.synchronize()
    T[name] = time.perf_counter() - t0
    return time.perf_counter()


W = {}


def warm(name, fn):
    """A device stage run a second time, synchronized: its time without the first
    call's allocations (reported beside the single-shot wall clock)."""
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    W[name] = time.perf_counter() - t
    return out


if "--reserve" in sys.argv:
    # one cached device block for every stage's buffers (see reserve_device_memory)
    from paper_1512_06235_b200 import reserve_device_memory
    reserve_device_memory(float(sys.argv[sys.argv.index("--reserve") + 1]))
t0 = time.perf_counter()
scene, snap = scenes.build(config, n_cameras=n_cam)
N = len(scene.cameras)
reg = set(int(i) for i in snap.registered)
queries = [i for i in range(N) if i not in reg]
nfeat = int(np.mean([len(fs) for fs in scene.feature_sets.values()]))
print(f"{config}: {N} cameras, {nfeat} features/img, M0 {len(reg)} cameras / "
      f"{len(snap.point_xyz)} points, {len(queries)} to localize", flush=True)
t0 = tick("scene (host synth)", t0)

# ---- 1. localization
S, n = scenes.track_sums(scene, snap)
pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
qbank = FeatureBank({q: scene.feature_sets[q] for q in queries})
dp = upload_points(pts, qbank.device)
t0 = tick("localize: query bank (host staging + H2D)", t0)
corrs = direct_search(qbank, pts, queries, device_points=dp)
t0 = tick("localize: kNN + ratio + direct search", t0)
warm("localize: kNN + ratio + direct search", lambda: direct_search(qbank, pts, queries, device_points=dp))
t0 = time.perf_counter()
todo = [k for k, c in enumerate(corrs) if len(c) > 16]
X = [snap.point_xyz[corrs[k][:, 0]] for k in todo]
uv = [scene.feature_sets[queries[k]].xy[corrs[k][:, 1]].astype(np.float64) for k in todo]
res = pnp_batch(X, uv, [scene.cameras[queries[k]].K for k in todo], [queries[k] for k in todo])
t0 = tick("localize: PnP-RANSAC", t0)
warm("localize: PnP-RANSAC", lambda: pnp_batch(X, uv, [scene.cameras[queries[k]].K for k in todo],
                                                [queries[k] for k in todo]))
t0 = time.perf_counter()
cams = {i: scene.cameras[i] for i in reg}
links = []                                   # (point row, image, fid) PnP inliers
rot_err = []
for k, r in zip(todo, res):
    if r.status != "ok":
        continue
    q = queries[k]
    cams[q] = Camera(K=scene.cameras[q].K, R=r.R, t=r.t, image_id=q)
    c = corrs[k][r.mask]
    links.append(np.stack([c[:, 0], np.full(len(c), q), c[:, 1]], 1))
    dR = r.R @ scene.cameras[q].R.T
    rot_err.append(np.degrees(np.arccos(np.clip((np.trace(dR) - 1) / 2, -1, 1))))
print(f"  localized {len(cams) - len(reg)}/{len(queries)}; median rotation error "
      f"{np.median(rot_err):.4f} deg", flush=True)

# ---- 2. M0 + the localized cameras' inliers as track observations
links = np.concatenate(links) if links else np.zeros((0, 3), np.int64)
owned = {i: snap.owned[i].copy() for i in snap.owned}
keep = []
for p_, q, f in links.tolist():
    if not owned[q][f]:
        owned[q][f] = True
        keep.append((p_, q, f))
keep = np.array(keep, np.int64).reshape(-1, 3)
old_pid = np.repeat(np.arange(len(snap.point_xyz)), np.diff(snap.track_ptr))
pid = np.concatenate([old_pid, keep[:, 0]])
img = np.concatenate([snap.track_img, keep[:, 1]]).astype(np.int32)
fid = np.concatenate([snap.track_fid, keep[:, 2]]).astype(np.int32)
order = np.lexsort((img, pid))
counts = np.bincount(pid, minlength=len(snap.point_xyz))
ptr = np.zeros(len(snap.point_xyz) + 1, np.int64)
np.cumsum(counts, out=ptr[1:])
snap1 = scenes.Snapshot(registered=np.array(sorted(cams), np.int64), point_xyz=snap.point_xyz,
                        track_ptr=ptr, track_img=img[order], track_fid=fid[order], owned=owned)
t0 = tick("register localized cameras", t0)

# ---- 3. densification over all registered cameras
pairs, qset = scenes.densify_pairs(snap1, N)
q_img, t_img, F = [], [], []
for a, b in pairs:
    q, t = (a, b) if a in qset else (b, a)
    try:
        F.append(fundamental_from_poses(cams[q], cams[t]).F)
    except DegenerateGeometryError:
        continue
    q_img.append(q)
    t_img.append(t)
imgs = sorted(set(q_img) | set(t_img))
untracked = {i: np.flatnonzero(~owned[i]).astype(np.int32) for i in imgs}
t0 = tick("densify: covisibility pairs + F", t0)
bank = FeatureBank(host=HostBank({i: scene.feature_sets[i] for i in imgs}))
t0 = tick("densify: bank H2D", t0)
mres = match_pairs(bank, np.array(q_img), np.array(t_img), np.stack(F),
                   [untracked[q] for q in q_img])
rows, n_matches = mres.packed()
t0 = tick("densify: geometry-aware matching", t0)
warm("densify: geometry-aware matching", lambda: match_pairs(
    bank, np.array(q_img), np.array(t_img), np.stack(F), [untracked[q] for q in q_img]).packed())
t0 = time.perf_counter()
qoff = torch.from_numpy(bank.offsets[[bank.index_of[q] for q in q_img]]).to(bank.device)
toff = torch.from_numpy(bank.offsets[[bank.index_of[t] for t in t_img]]).to(bank.device)
pk = rows[:, 0].long()
u = (qoff[pk] + (rows[:, 1] & 0xFFFF).long()).to(torch.int32).contiguous()
v = (toff[pk] + ((rows[:, 1] >> 16) & 0xFFFF).long()).to(torch.int32).contiguous()
dist = rows[:, 2].contiguous().view(torch.float32)
in_bank = np.isin(snap1.track_img, imgs)
slot = np.array([bank.index_of.get(int(i), 0) for i in snap1.track_img], np.int64)
tnode = (bank.offsets[slot] + snap1.track_fid)[in_bank].astype(np.int32)
tptr = np.zeros(len(snap1.point_xyz) + 1, np.int64)
np.cumsum(np.bincount(np.repeat(np.arange(len(snap1.point_xyz)), np.diff(snap1.track_ptr))[in_bank],
                      minlength=len(snap1.point_xyz)), out=tptr[1:])
nodes, owners, offs = merge_tracks_nodes(bank, u, v, dist, tptr, tnode)
t0 = tick("densify: track merge", t0)
warm("densify: track merge", lambda: merge_tracks_nodes(bank, u, v, dist, tptr, tnode))
t0 = time.perf_counter()
# tracks to triangulate: new tracks, and grown tracks with their existing refs (vectorized)
cam_ids = sorted(cams)
cam_of_img = np.full(N, -1, np.int64)
cam_of_img[cam_ids] = np.arange(len(cam_ids))
slot_n = np.searchsorted(bank.offsets, nodes, "right") - 1
node_img = np.array(bank.image_ids, np.int64)[slot_n]
node_fid = nodes - bank.offsets[slot_n]
seg_len = np.diff(offs)
own = owners.astype(np.int64)
ex_len = np.where(own >= 0, np.diff(snap1.track_ptr)[np.maximum(own, 0)], 0)
tot_len = seg_len + ex_len
trk_ptr = np.zeros(len(own) + 1, np.int64)
np.cumsum(tot_len, out=trk_ptr[1:])
trk_img = np.empty(int(trk_ptr[-1]), np.int64)
trk_fid = np.empty(int(trk_ptr[-1]), np.int64)
# existing refs first, then the fresh nodes, per segment
seg_of_ex = np.repeat(np.arange(len(own)), ex_len)
ex_rank = np.arange(len(seg_of_ex)) - np.repeat(np.cumsum(ex_len) - ex_len, ex_len)
ex_src = snap1.track_ptr[np.maximum(own, 0)][seg_of_ex] + ex_rank
ex_dst = trk_ptr[seg_of_ex] + ex_rank
trk_img[ex_dst] = snap1.track_img[ex_src]
trk_fid[ex_dst] = snap1.track_fid[ex_src]
seg_of_fr = np.repeat(np.arange(len(own)), seg_len)
fr_dst = trk_ptr[seg_of_fr] + ex_len[seg_of_fr] + (np.arange(len(nodes)) - offs[seg_of_fr])
trk_img[fr_dst] = node_img
trk_fid[fr_dst] = node_fid
all_off = np.zeros(N + 1, np.int64)
np.cumsum([len(scene.feature_sets[i]) for i in range(N)], out=all_off[1:])
all_xy = np.concatenate([scene.feature_sets[i].xy for i in range(N)])
hxy = all_xy[all_off[trk_img] + trk_fid]
trk_kind = own < 0
t0 = tick("densify: track assembly (host)", t0)
K = np.stack([cams[c].K for c in cam_ids]); R = np.stack([cams[c].R for c in cam_ids])
tt = np.stack([cams[c].t for c in cam_ids])
st, Xt, err = triangulate_batch(K, R, tt, trk_ptr, cam_of_img[trk_img].astype(np.int32),
                                hxy.astype(np.float64))
t0 = tick("densify: triangulation", t0)
warm("densify: triangulation", lambda: triangulate_batch(K, R, tt, trk_ptr, cam_of_img[trk_img].astype(np.int32),
                                                         hxy.astype(np.float64)))
kind = np.array(trk_kind, bool)
new_ok = int(((st == 1) & kind).sum())
ext_ok = int(((st == 1) & ~kind).sum())
# accuracy of the new points against the ground truth world points
gt_err = []
for s_ in np.flatnonzero((st == 1) & kind)[:20000]:
    sel = slice(offs[s_], offs[s_ + 1])
    wp = {int(scene.point_of_feature[int(i_)][int(f_)]) for i_, f_ in zip(node_img[sel], node_fid[sel])}
    if len(wp) == 1 and -1 not in wp:
        gt_err.append(np.linalg.norm(Xt[s_] - scene.points[wp.pop()]))
print(f"  pairs {len(q_img)}, matches {n_matches}, new tracks {int(kind.sum())} "
      f"({new_ok} triangulated), grown tracks {int((~kind).sum())} ({ext_ok} re-triangulated); "
      f"new-point error vs ground truth: median {np.median(gt_err):.4f}, "
      f"{100 * np.mean(np.array(gt_err) < 0.05):.1f}% < 0.05 (scene units, {len(gt_err)} points)")
print(f"  {'stage':42s} {'first call':>10s} {'warm':>9s}   (wall clock, device synchronized)")
for k_, v_ in T.items():
    w_ = f"{1e3 * W[k_]:9.1f}" if k_ in W else f"{'':9s}"
    print(f"  {k_:42s} {1e3 * v_:10.1f} {w_} ms")
