"""Benchmark/parity workloads C1-C5 as flat host arrays.

Builds, from a seeded synthetic scene, exactly the inputs the reference's
fine stages see:

* the coarse model M0 (GT poses of the registered cameras; GT points restricted
  to coarse-tier refs ``fid < coarse_count`` at eta=20 with >= 2 refs, point
  ids assigned in ascending GT point order) — SURVEY.md Appendix B;
* densify's pair list: ``candidate_images`` (densify.py:37-56) for every
  registered image, ``unique_pairs`` (densify.py:59-65), query/target roles
  (densify.py:222) and the untracked query lists (densify.py:199-207);
* for localization, the point list with its track CSR (pid -> (image, fid)).

Covisibility is a sparse product V·Vᵀ instead of the reference's per-pair
Python set intersections (same counts, same ordering rules).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .geometry import fundamental_from_poses
from .synth import SceneSpec, generate_scene
from .types import DegenerateGeometryError, FeatureRef, Model

COVIS_THRESHOLD = 8
CANDIDATE_FRACTION = 0.10


@dataclass
class Snapshot:
    """Read-only coarse model flattened to arrays."""

    registered: np.ndarray          # sorted image ids with a pose
    point_xyz: np.ndarray           # (M, 3) f64, row = point id
    track_ptr: np.ndarray           # (M+1,) int64 CSR over observations
    track_img: np.ndarray           # (nobs,) int32, ascending image id within a track
    track_fid: np.ndarray           # (nobs,) int32
    owned: dict                     # image id -> bool (n_i,) feature owned by a point


def tier_counts(sets: dict, eta: float = 20.0) -> dict:
    """select_top_scale (features.py:149-161) applied to every image."""
    out = {}
    for i, fs in sets.items():
        n = len(fs)
        out[i] = n if n < 1000 else math.ceil(eta / 100.0 * n)
    return out


def coarse_snapshot(scene, registered, eta: float | None = 20.0) -> Snapshot:
    """GT points restricted to the registered cameras' refs (and to each image's
    coarse tier when eta is given), >= 2 refs, ids in ascending GT order."""
    registered = np.array(sorted(int(i) for i in registered), dtype=np.int64)
    reg_mask = np.zeros(len(scene.cameras), dtype=bool)
    reg_mask[registered] = True
    tiers = tier_counts(scene.feature_sets, eta if eta is not None else 100.0)
    n_pts = len(scene.points)
    # observation table of every (image, fid) that sees a world point
    obs_img, obs_fid, obs_pid = [], [], []
    for i in sorted(scene.feature_sets):
        pof = scene.point_of_feature[i]
        f = np.flatnonzero(pof >= 0)
        obs_img.append(np.full(len(f), i, np.int64)); obs_fid.append(f); obs_pid.append(pof[f])
    obs_img = np.concatenate(obs_img); obs_fid = np.concatenate(obs_fid)
    obs_pid = np.concatenate(obs_pid)
    # triangulable = seen in >= 2 images (GT model membership, synth.py:86-116)
    seen = np.bincount(obs_pid, minlength=n_pts)
    tier_arr = np.array([tiers.get(i, 0) if eta is not None else 1 << 40
                         for i in range(len(scene.cameras))], dtype=np.int64)
    tier_of = tier_arr[obs_img]
    keep = reg_mask[obs_img] & (obs_fid < tier_of) & (seen[obs_pid] >= 2)
    k_img, k_fid, k_pid = obs_img[keep], obs_fid[keep], obs_pid[keep]
    kept_per_pid = np.bincount(k_pid, minlength=n_pts)
    good = kept_per_pid >= 2
    sel = good[k_pid]
    k_img, k_fid, k_pid = k_img[sel], k_fid[sel], k_pid[sel]
    order = np.lexsort((k_img, k_pid))
    k_img, k_fid, k_pid = k_img[order], k_fid[order], k_pid[order]
    gt_ids = np.flatnonzero(good)                # ascending GT ids -> model ids 0..M-1
    remap = np.full(n_pts, -1, np.int64)
    remap[gt_ids] = np.arange(len(gt_ids))
    counts = np.bincount(remap[k_pid], minlength=len(gt_ids))
    ptr = np.zeros(len(gt_ids) + 1, np.int64)
    np.cumsum(counts, out=ptr[1:])
    owned = {i: np.zeros(len(scene.feature_sets[i]), dtype=bool) for i in scene.feature_sets}
    by_img = np.argsort(k_img, kind="stable")
    bounds = np.searchsorted(k_img[by_img], np.arange(len(scene.cameras) + 1))
    for i in sorted(scene.feature_sets):
        owned[i][k_fid[by_img[bounds[i]:bounds[i + 1]]]] = True
    return Snapshot(registered=registered, point_xyz=scene.points[gt_ids].copy(),
                    track_ptr=ptr, track_img=k_img.astype(np.int32),
                    track_fid=k_fid.astype(np.int32), owned=owned)


def snapshot_to_model(scene, snap: Snapshot) -> Model:
    """The same snapshot as a ``Model`` (for the per-call drop-in API)."""
    model = Model(stage_tag="coarse")
    for i in snap.registered:
        model.attach_camera(scene.cameras[int(i)])
    for p in range(len(snap.point_xyz)):
        lo, hi = snap.track_ptr[p], snap.track_ptr[p + 1]
        model.add_point(snap.point_xyz[p], [FeatureRef(int(i), int(f)) for i, f in
                                            zip(snap.track_img[lo:hi], snap.track_fid[lo:hi])])
    return model


def covisibility(snap: Snapshot, n_images: int) -> np.ndarray:
    """(N, N) shared-point counts == len(model.covisible_points(a, b))."""
    M = len(snap.point_xyz)
    V = np.zeros((n_images, M), dtype=np.float32)
    pid = np.repeat(np.arange(M), np.diff(snap.track_ptr))
    V[snap.track_img, pid] = 1.0
    C = (V @ V.T).astype(np.int64)   # exact: counts < 2^24
    return C


def densify_pairs(snap: Snapshot, n_images: int, query_images=None,
                  threshold: int = COVIS_THRESHOLD,
                  candidate_fraction: float = CANDIDATE_FRACTION):
    """Sorted unique pairs (densify.py:186-196) and the query set."""
    reg = [int(i) for i in snap.registered]
    if query_images is None:
        query_images = reg
    reg_set = set(reg)
    query_images = [i for i in sorted(query_images) if i in reg_set]
    k_limit = max(1, int(np.ceil(candidate_fraction * len(reg))))
    C = covisibility(snap, n_images)
    pairs = set()
    for i in query_images:
        scored = sorted((-int(C[i, o]), o) for o in reg if o != i and C[i, o] > threshold)
        for _, o in scored[:k_limit]:
            pairs.add((i, o) if i < o else (o, i))
    return sorted(pairs), set(query_images)


@dataclass
class PairWorkload:
    """Everything one densify pass hands the matcher, in pair order."""

    pairs: list            # sorted (a, b)
    q_img: np.ndarray      # (P,) query image per pair
    t_img: np.ndarray      # (P,) target image per pair
    F: np.ndarray          # (P, 3, 3) f64 (rows for degenerate pairs are NaN and skipped)
    valid: np.ndarray      # (P,) bool: F defined
    untracked: dict        # image id -> sorted int32 untracked feature ids


def pair_workload(scene, snap: Snapshot, query_images=None) -> PairWorkload:
    pairs, qset = densify_pairs(snap, len(scene.cameras), query_images)
    P = len(pairs)
    q_img = np.zeros(P, np.int32); t_img = np.zeros(P, np.int32)
    F = np.full((P, 3, 3), np.nan); valid = np.zeros(P, bool)
    for k, (a, b) in enumerate(pairs):
        q, t = (a, b) if a in qset else (b, a)
        q_img[k], t_img[k] = q, t
        try:
            F[k] = fundamental_from_poses(scene.cameras[q], scene.cameras[t]).F
            valid[k] = True
        except DegenerateGeometryError:
            pass
    imgs = sorted({x for p in pairs for x in p})
    untracked = {i: np.flatnonzero(~snap.owned[i]).astype(np.int32) for i in imgs}
    return PairWorkload(pairs=pairs, q_img=q_img, t_img=t_img, F=F, valid=valid,
                        untracked=untracked)


# ---------------------------------------------------------------- configs ---

def spec_for(config: str, n_cameras: int | None = None) -> SceneSpec:
    """SceneSpec of a named config."""
    if config == "C1":
        return SceneSpec(n_cameras=n_cameras or 20, n_points=2000, visibility_fraction=0.6,
                         pixel_noise=0.5, descriptor_noise=4.0, seed=1)
    if config in ("C2", "C3"):
        return SceneSpec(n_cameras=n_cameras or (100 if config == "C2" else 320),
                         n_points=12000, image_width=3072, image_height=2304, focal=2600.0,
                         visibility_fraction=0.55, clutter_per_image=2700, pixel_noise=0.5,
                         descriptor_noise=4.0, seed=2)
    if config in ("C4", "C5"):
        return SceneSpec(n_cameras=n_cameras or (500 if config == "C4" else 3000),
                         n_points=24000, image_width=3072, image_height=2304, focal=2600.0,
                         visibility_fraction=0.55, clutter_per_image=5400, pixel_noise=0.5,
                         descriptor_noise=4.0, seed=4)
    raise ValueError(f"unknown config {config!r}")


def registered_for(config: str, n_cameras: int) -> list:
    if config in ("C1", "C3"):
        return list(range(n_cameras))
    return list(range(0, n_cameras, 5))


def build(config: str, n_cameras: int | None = None):
    spec = spec_for(config, n_cameras)
    scene = generate_scene(spec)
    snap = coarse_snapshot(scene, registered_for(config, spec.n_cameras))
    return scene, snap


def track_sums(scene, snap: Snapshot):
    """Per point: S = sum of track descriptors (int32, <= 255*n) and n = track
    length — the exact form of mean_descriptor (localize.py:51-59)."""
    M = len(snap.point_xyz)
    S = np.zeros((M, 128), dtype=np.int64)
    pid = np.repeat(np.arange(M), np.diff(snap.track_ptr))
    for i in np.unique(snap.track_img):
        sel = np.flatnonzero(snap.track_img == i)
        np.add.at(S, pid[sel], scene.feature_sets[int(i)].descriptors[snap.track_fid[sel]].astype(np.int64))
    n = np.diff(snap.track_ptr).astype(np.int32)
    return S.astype(np.int32), n
