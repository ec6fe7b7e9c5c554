"""3D-2D localization on the device: kNN (tcgen05) -> ratio/dedupe -> PnP-RANSAC.

Batched API ``direct_search`` (one call for all query images of a stage) plus
reference-shaped drop-ins (``direct_3d2d_search``, ``localize_image``,
``localize_all``; localize.py:99-281 of the reference).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from .bank import FeatureBank
from .types import LocalizationResult, SetCover

RATIO_UNGUIDED = 0.6     # matching.py:21
SINGLE_CANDIDATE_CAP = 45.0
MIN_CORRESPONDENCES = 16  # localize.py:30
KEY_BIG = 0x7FFFFFFFFFFFFFFF      # no second neighbour (msfm_knn2_tracks)


def ratio_fraction(ratio: float):
    f = Fraction(float(ratio)).limit_denominator(1 << 20)
    return f.numerator, f.denominator


@dataclass
class PointSet:
    """Exact query points: track sums S (M,128) int32, lengths n (M,), ids.
    ``dev``: (S, n, |S|^2) already on the device (track_sums_device); S is then
    None on the host until someone asks for it."""

    S: np.ndarray
    n: np.ndarray
    ids: np.ndarray
    dev: tuple = None

    @property
    def SS(self) -> np.ndarray:
        """|S|^2 per point (int64), computed once."""
        ss = self.__dict__.get("_ss")
        if ss is None or len(ss) != len(self.n):
            if self.S is None:
                ss = self.dev[2][:len(self.n)].cpu().numpy().astype(np.int64)
            else:
                S = self.S.astype(np.int64)
                ss = (S * S).sum(1)
            self.__dict__["_ss"] = ss
        return ss


def track_sums_device(bank: FeatureBank, track_ptr, track_row, stream=None):
    """K7 (mean_descriptor localize.py:51-59, exact integer form) on the device:
    point p's track is bank rows track_row[track_ptr[p]:track_ptr[p+1]].  Returns
    (S int32 (M,128), n int32 (M,), |S|^2 int64 (M,)) device tensors."""
    import torch

    lib = _lib.load()
    dev = bank.device
    ptr = np.ascontiguousarray(track_ptr, np.int64)
    M = len(ptr) - 1
    d_ptr = _lib.h2d(ptr, dev)
    d_row = _lib.h2d(np.ascontiguousarray(track_row, np.int64) if len(track_row) else
                     np.zeros(1, np.int64), dev)
    dS = torch.empty((max(M, 1), 128), dtype=torch.int32, device=dev)
    dn = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
    dSS = torch.empty(max(M, 1), dtype=torch.int64, device=dev)
    b = bank.cstruct()
    _lib.check(lib.msfm_track_sums(ctypes.byref(b), M, _lib.ptr(d_ptr), _lib.ptr(d_row),
                                   _lib.ptr(dS), _lib.ptr(dn), _lib.ptr(dSS),
                                   _lib.stream_handle(stream)), "msfm_track_sums")
    return dS, dn, dSS


def points_from_snapshot(scene_sets, snap, ids=None) -> PointSet:
    from .scenes import track_sums

    class _Scene:
        feature_sets = scene_sets

    S, n = track_sums(_Scene, snap)
    ids = np.arange(len(S)) if ids is None else np.asarray(ids)
    return PointSet(S=S[ids], n=n[ids], ids=ids)


@dataclass
class DeviceKnn:
    k1: object
    i1: object
    k2: object
    M_pad: int
    keep: tuple = field(default=())
    i2: object = None          # second neighbour's index (knn2_tracks(second=True))

    def host_all(self, pts: PointSet):
        """(idx, N_best, N_second) of every query slot: (S, M) arrays, three copies."""
        M = len(pts.n)
        k1 = self.k1[:, :M].cpu().numpy().astype(np.int64)
        i1 = self.i1[:, :M].cpu().numpy().astype(np.int64)
        k2 = self.k2[:, :M].cpu().numpy().astype(np.int64)
        n = pts.n.astype(np.int64)[None, :]
        SS = pts.SS[None, :]
        Nb = n * k1 + SS
        Ns = np.where(k2 == KEY_BIG, -1, n * np.where(k2 == KEY_BIG, 0, k2) + SS)
        return i1, Nb, Ns

    def host(self, pts: PointSet, s: int):
        """(idx, N_best, N_second) of query slot s, N_second=-1 if undefined."""
        M = len(pts.n)
        k1 = self.k1[s, :M].cpu().numpy().astype(np.int64)
        i1 = self.i1[s, :M].cpu().numpy().astype(np.int64)
        k2 = self.k2[s, :M].cpu().numpy().astype(np.int64)
        n = pts.n.astype(np.int64)
        SS = pts.SS
        Nb = n * k1 + SS
        Ns = np.where(k2 == KEY_BIG, -1, n * np.where(k2 == KEY_BIG, 0, k2) + SS)
        return i1, Nb, Ns


def knn2_tracks(bank: FeatureBank, pts: PointSet, image_ids, stream=None,
                device_points=None, counts=None, second: bool = False, into=None) -> DeviceKnn:
    """Top-2 over each image's features; ``counts`` (per bank image, optional)
    restricts image k to its first counts[k] features (a coarse tier); ``second``
    also resolves the second neighbour's index (lowest index at the second key)."""
    import torch

    lib = _lib.load()
    M = len(pts.n)
    M_pad = (M + 127) // 128 * 128
    dev = bank.device
    if device_points is None:
        device_points = upload_points(pts, dev)
    dS, dn, dSS = device_points
    slots = np.array([bank.index_of[int(i)] for i in image_ids], dtype=np.int32)
    d_slots = _lib.h2d(slots, dev)
    if into is not None:
        # (k1, i1, k2) rows of these images inside larger tables (row views)
        k1, i1, k2 = into
    else:
        k1 = torch.empty((max(len(slots), 1), M_pad), dtype=torch.int64, device=dev)
        i1 = torch.empty((max(len(slots), 1), M_pad), dtype=torch.int32, device=dev)
        k2 = torch.empty_like(k1)
    cnt = bank.counts if counts is None else np.asarray(counts, np.int64)
    max_feat = int(cnt[slots].max()) if len(slots) else 0
    ws_bytes = lib.msfm_knn_workspace_bytes(M, len(slots), max_feat)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    b = bank.cstruct()
    d_cnt = None
    if counts is not None:
        d_cnt = _lib.h2d(cnt.astype(np.int32), dev)
        b.d_img_n = _lib.ptr(d_cnt)
    maxn = int(pts.n.max()) if M else 0
    _lib.check(lib.msfm_knn2_tracks(ctypes.byref(b), M, _lib.ptr(dS), _lib.ptr(dn), len(slots),
                                    _lib.ptr(d_slots), maxn, max_feat, _lib.ptr(k1), _lib.ptr(i1),
                                    _lib.ptr(k2), _lib.ptr(ws), ws_bytes,
                                    _lib.stream_handle(stream)), "msfm_knn2_tracks")
    out = DeviceKnn(k1, i1, k2, M_pad, keep=(ws, d_slots, d_cnt))
    if second:
        out.i2 = torch.empty_like(i1)
        _lib.check(lib.msfm_knn2_second_index(ctypes.byref(b), M, _lib.ptr(dS), _lib.ptr(dn),
                                              len(slots), _lib.ptr(d_slots), _lib.ptr(k1),
                                              _lib.ptr(i1), _lib.ptr(k2), _lib.ptr(out.i2),
                                              _lib.stream_handle(stream)),
                   "msfm_knn2_second_index")
    return out


def knn2_tracks_staged(bank: FeatureBank, pts: PointSet, image_ids, device_points,
                       groups: int = 8) -> DeviceKnn:
    """knn2_tracks on a staged bank (FeatureBank(staged=True)) whose rows are
    still in pinned host memory: the images go up in ``groups`` contiguous ranges
    on a copy stream, and the kNN of range g (with its |desc|^2) runs as soon as
    it has landed, while range g + 1 is in flight.  ``image_ids`` must be the
    bank's images in bank order."""
    import torch

    lib = _lib.load()
    dev = bank.device
    ids = list(image_ids)
    S = len(ids)
    assert list(bank.slots(ids)) == list(range(S)), "image_ids must be the bank's images in order"
    M_pad = (len(pts.n) + 127) // 128 * 128
    k1 = torch.empty((max(S, 1), M_pad), dtype=torch.int64, device=dev)
    i1 = torch.empty((max(S, 1), M_pad), dtype=torch.int32, device=dev)
    k2 = torch.empty_like(k1)
    cs = bank.__dict__.get("_h2d_stream")
    if cs is None:
        cs = bank.__dict__["_h2d_stream"] = torch.cuda.Stream(device=dev)
    cur = torch.cuda.current_stream(dev)
    cs.wait_stream(cur)
    if not bank.__dict__.get("_recorded"):
        # the rows are written on `cs`: the allocator must not recycle them early
        bank.xy.record_stream(cs)
        bank.desc.record_stream(cs)
        bank.__dict__["_recorded"] = True
    edges = np.linspace(0, S, max(1, min(groups, S)) + 1).round().astype(int)
    keep = []
    for g0, g1 in zip(edges[:-1], edges[1:]):
        if g1 <= g0:
            continue
        landed = bank.upload_range(int(g0), int(g1), cs)
        cur.wait_event(landed)
        a, b = bank.row_range(int(g0), int(g1))
        _lib.check(lib.msfm_feature_norms(_lib.ptr(bank.desc) + 128 * a, b - a,
                                          _lib.ptr(bank.norm2) + 4 * a, _lib.stream_handle(cur)),
                   "msfm_feature_norms")
        keep.append(knn2_tracks(bank, pts, ids[g0:g1], device_points=device_points,
                                into=(k1[g0:g1], i1[g0:g1], k2[g0:g1])))
    return DeviceKnn(k1, i1, k2, M_pad, keep=tuple(keep))


def upload_points(pts: PointSet, dev):
    """(S, n, |S|^2) on the device; the pinned host copies are made once per
    PointSet, so repeated uploads are three async copies."""
    import torch

    if pts.dev is not None:
        return pts.dev
    pinned = pts.__dict__.get("_pinned")
    if pinned is None or pinned[0] is not pts.S:
        M = len(pts.n)

        def pin(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()

        pinned = (pts.S, pin(pts.S.astype(np.int32) if M else np.zeros((1, 128), np.int32)),
                  pin(pts.n.astype(np.int32) if M else np.zeros(1, np.int32)),
                  pin(pts.SS if M else np.zeros(1, np.int64)))
        pts.__dict__["_pinned"] = pinned
    return tuple(t.to(dev, non_blocking=True) for t in pinned[1:])


@dataclass
class Correspondences:
    """Per query image: (point row, feature id) sorted by point row."""

    rows: object
    fids: object
    counts: object
    M_pad: int

    def get(self, s: int):
        c = int(self.counts[s])
        return self.rows[s, :c], self.fids[s, :c]


def direct_search(bank: FeatureBank, pts: PointSet, image_ids, *, ratio: float = RATIO_UNGUIDED,
                  single_cap: float = SINGLE_CANDIDATE_CAP, stream=None, device_points=None,
                  knn: DeviceKnn | None = None, to_host: bool = True, flat: bool = False,
                  device_flat: bool = False):
    """direct_3d2d_search for many images: kNN + ratio + one point per feature."""
    import torch

    lib = _lib.load()
    dev = bank.device
    if device_points is None:
        device_points = upload_points(pts, dev)
    if knn is None:
        knn = knn2_tracks(bank, pts, image_ids, stream, device_points)
    dS, dn, dSS = device_points
    M = len(pts.n)
    slots = np.array([bank.index_of[int(i)] for i in image_ids], dtype=np.int32)
    d_slots = _lib.h2d(slots, dev)
    nfeat = bank.counts[slots].astype(np.int64)
    win_off = np.zeros(len(slots), np.int64)
    if len(slots) > 1:
        np.cumsum(nfeat[:-1], out=win_off[1:])
    d_win_off = _lib.h2d(win_off, dev)
    win = torch.empty(max(int(nfeat.sum()), 1), dtype=torch.int32, device=dev)
    rows = torch.empty((max(len(slots), 1), knn.M_pad), dtype=torch.int32, device=dev)
    fids = torch.empty_like(rows)
    cnt = torch.zeros(max(len(slots), 1), dtype=torch.int32, device=dev)
    p, q = ratio_fraction(ratio)
    b = bank.cstruct()
    _lib.check(lib.msfm_direct_3d2d(ctypes.byref(b), M, _lib.ptr(dn), _lib.ptr(dSS), len(slots),
                                    _lib.ptr(d_slots), _lib.ptr(knn.k1), _lib.ptr(knn.i1),
                                    _lib.ptr(knn.k2), p, q, float(single_cap), _lib.ptr(win),
                                    _lib.ptr(d_win_off), _lib.ptr(rows), _lib.ptr(fids),
                                    _lib.ptr(cnt), _lib.stream_handle(stream)), "msfm_direct_3d2d")
    res = Correspondences(rows, fids, cnt, knn.M_pad)
    res._keep = (win, d_win_off, d_slots, knn)
    if device_flat:
        # (point rows, feature ids) on the device, offsets on the host: image s owns
        # [off[s], off[s+1]); one small copy (the counts)
        c = cnt[:len(slots)].cpu().numpy()
        off = np.zeros(len(slots) + 1, np.int64)
        np.cumsum(c, out=off[1:])
        keep = torch.arange(knn.M_pad, device=dev)[None, :] < cnt[:len(slots), None]
        return rows[:len(slots)][keep].long(), fids[:len(slots)][keep].long(), off
    if to_host:
        # three copies in total (counts, then the used prefix of both tables)
        c = cnt.cpu().numpy()
        w = int(c.max()) if len(c) else 0
        rh = rows[:, :w].cpu().numpy()
        fh = fids[:, :w].cpu().numpy()
        if flat:
            # (point ids, feature ids, offsets): image s owns [off[s], off[s+1])
            off = np.zeros(len(slots) + 1, np.int64)
            np.cumsum(c[:len(slots)], out=off[1:])
            keep = np.arange(w)[None, :] < c[:len(slots), None]
            return pts.ids[rh[keep]].astype(np.int64), fh[keep].astype(np.int64), off
        return [np.stack([pts.ids[rh[s, :c[s]]], fh[s, :c[s]]], 1).astype(np.int64)
                for s in range(len(slots))]
    return res


def gather_pnp_inputs(bank: FeatureBank, corr: Correspondences, image_ids, d_xyz,
                      gate: int = MIN_CORRESPONDENCES, stream=None):
    """The PnP inputs of the images with more than ``gate`` correspondences
    (localize.py:203-211) straight from ``direct_search(to_host=False)``: X (N, 3)
    and uv (N, 2) f64 on the device (msfm_gather_3d2d, one launch), per-image
    offsets (host) and the selected positions in ``image_ids``.  One small copy
    each way (the counts back, the selection out)."""
    import torch

    lib = _lib.load()
    dev = bank.device
    B = len(image_ids)
    c = corr.counts[:B].cpu().numpy().astype(np.int64)
    todo = np.flatnonzero(c > gate)
    off = np.zeros(len(todo) + 1, np.int64)
    np.cumsum(c[todo], out=off[1:])
    N = int(off[-1])
    row0 = bank.offsets[bank.slots(np.asarray(image_ids)[todo])] if len(todo) else \
        np.zeros(0, np.int64)
    meta = torch.from_numpy(np.concatenate([todo.astype(np.int64), row0, off])).pin_memory()
    d_meta = meta.to(dev, non_blocking=True)
    k = len(todo)
    X = torch.empty((max(N, 1), 3), dtype=torch.float64, device=dev)
    uv = torch.empty((max(N, 1), 2), dtype=torch.float64, device=dev)
    base = _lib.ptr(d_meta)
    _lib.check(lib.msfm_gather_3d2d(_lib.ptr(corr.rows), _lib.ptr(corr.fids), corr.M_pad, k, base,
                                    base + 8 * k, base + 16 * k, _lib.ptr(d_xyz),
                                    _lib.ptr(bank.xy), _lib.ptr(X), _lib.ptr(uv),
                                    _lib.stream_handle(stream)), "msfm_gather_3d2d")
    return X[:N], uv[:N], off, todo


# ---------------------------------------------------------------------------
# reference-shaped stage API (localize.py:33-281)
# ---------------------------------------------------------------------------

SET_COVER_K = 400
SET_COVER_ENGAGE_POINTS = 100_000
RANKED_TOP_K = 10


def compute_set_cover(model, k: int = SET_COVER_K) -> SetCover:
    """k-cover of the cameras by points (localize.py:62-96): repeatedly take the
    point that sees the most cameras still short of k views; ties go to the
    longer track, then to the lower point id; stop when every camera has k views
    or no point adds any.  Host side, off the per-image path.

    Restated over arrays: the tracks become a CSR of camera slots with its
    slot -> points inverse, and every point's score is a counter that drops by
    one when a camera it sees reaches k (scores only fall).  A bucket queue
    indexed by score, each bucket a heap of static (-length, id) ranks, yields
    the argmax: entries whose score went stale are moved to their current
    bucket when they surface."""
    import heapq

    if k < 1:
        raise ValueError(f"coverage target must be >= 1, got {k}")
    cams = list(model.cameras)
    pids = np.array(sorted(model.points), dtype=np.int64)
    tracks = [list(model.points[int(p)].track) for p in pids]
    lens = np.fromiter((len(t) for t in tracks), np.int64, len(tracks))
    ptr = np.zeros(len(pids) + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    img = np.fromiter((i for t in tracks for i in t), np.int64, int(ptr[-1]))
    cam_ids = np.array(cams, dtype=np.int64)
    slot = np.full(len(img), -1, np.int64)
    if len(cams):
        srt = np.argsort(cam_ids, kind="stable")
        pos = np.minimum(np.searchsorted(cam_ids[srt], img), len(cams) - 1)
        hit = cam_ids[srt][pos] == img
        slot[hit] = srt[pos[hit]]
    owner = np.repeat(np.arange(len(pids)), lens)
    seen = slot >= 0
    score = np.bincount(owner[seen], minlength=len(pids)).astype(np.int64)
    by_slot = np.argsort(slot[seen], kind="stable")
    obs_owner = owner[seen][by_slot]
    obs_ptr = np.searchsorted(slot[seen][by_slot], np.arange(len(cams) + 1))
    rank_order = np.lexsort((pids, -lens))          # rank r -> point index
    top = int(score.max()) if len(pids) else 0
    buckets = [[] for _ in range(top + 1)]
    for r, p in enumerate(rank_order):              # ascending ranks: each list is a heap
        if score[p] > 0:
            buckets[score[p]].append(r)
    remaining = np.full(len(cams), k, np.int64)
    unsaturated = len(cams)
    selected = []
    while top > 0 and unsaturated > 0:
        if not buckets[top]:
            top -= 1
            continue
        r = heapq.heappop(buckets[top])
        p = rank_order[r]
        s = int(score[p])
        if s != top:
            if s > 0:
                heapq.heappush(buckets[s], r)
            continue
        selected.append(int(pids[p]))
        sl = slot[ptr[p]:ptr[p + 1]]
        sl = sl[sl >= 0]
        sl = sl[remaining[sl] > 0]
        remaining[sl] -= 1
        for c in sl[remaining[sl] == 0]:
            score[obs_owner[obs_ptr[c]:obs_ptr[c + 1]]] -= 1
            unsaturated -= 1
    coverage = {i: 0 for i in cams}
    sel_idx = np.searchsorted(pids, np.array(selected, dtype=np.int64))
    if len(sel_idx):
        per = np.concatenate([slot[ptr[p]:ptr[p + 1]] for p in sel_idx])
        counts = np.bincount(per[per >= 0], minlength=len(cams))
        for j, i in enumerate(cams):
            coverage[i] = int(counts[j])
        if (per < 0).any():                         # track images without a camera
            for p in sel_idx:
                for i, c in zip(tracks[p], slot[ptr[p]:ptr[p + 1]]):
                    if c < 0:
                        coverage[i] = coverage.get(i, 0) + 1
    return SetCover(selected=selected, k=k, coverage=coverage)


def model_points(model, feature_store, point_ids) -> PointSet:
    """Exact track sums of the listed points (mean_descriptor, localize.py:51-59):
    the tracks flattened to a CSR over a device bank of their images, summed by
    the K7 kernel (msfm_track_sums) on the device."""
    from itertools import chain

    pids = np.asarray(sorted(point_ids), dtype=np.int64)
    tracks = [model.points[int(p)].track for p in pids]
    n = np.fromiter((len(t) for t in tracks), np.int64, len(tracks))
    ptr = np.zeros(len(pids) + 1, np.int64)
    np.cumsum(n, out=ptr[1:])
    total = int(ptr[-1])
    imgs = np.fromiter(chain.from_iterable(t.keys() for t in tracks), np.int64, total)
    fids = np.fromiter(chain.from_iterable(t.values() for t in tracks), np.int64, total)
    used = sorted(set(imgs.tolist()))
    bank = FeatureBank({int(i): feature_store.sets[int(i)] for i in used}) if used else None
    if bank is None:
        return PointSet(S=np.zeros((len(pids), 128), np.int32), n=n.astype(np.int32), ids=pids)
    slot = np.array([bank.index_of[int(i)] for i in used], np.int64)
    lut = dict(zip(used, bank.offsets[slot].tolist()))
    base = np.fromiter((lut[i] for i in imgs.tolist()), np.int64, total)
    dS, dn, dSS = track_sums_device(bank, ptr, base + fids)
    pts = PointSet(S=None, n=n.astype(np.int32), ids=pids, dev=(dS, dn, dSS))
    pts.__dict__["_track_bank"] = bank        # keeps the rows alive with the sums
    return pts


def direct_3d2d_search(model, point_ids, image_fs, feature_store, *, ratio=RATIO_UNGUIDED,
                       single_cap=SINGLE_CANDIDATE_CAP, index=None, stats=None):
    """Drop-in for localize.py:99-122 (exact kNN on the device)."""
    pids = sorted(point_ids)
    if not pids or len(image_fs) == 0:
        return []
    pts = model_points(model, feature_store, pids)
    bank = FeatureBank({int(image_fs.image_id): image_fs})
    if stats is not None:
        stats.add(len(pids), len(pids) * len(image_fs))
    corr = direct_search(bank, pts, [int(image_fs.image_id)], ratio=ratio, single_cap=single_cap)[0]
    return [(int(p), int(f)) for p, f in corr]


def _knn_u8(bank, image_id, queries_u8):
    """knn2 of u8 query descriptors (track length 1): exact f32 distances as the
    reference computes them (descriptors.py:55-69, all partials < 2^24)."""
    q = np.asarray(queries_u8, dtype=np.int32).reshape(-1, 128)
    pts = PointSet(S=q, n=np.ones(len(q), np.int32), ids=np.arange(len(q)))
    res = knn2_tracks(bank, pts, [image_id])
    idx, nb, ns = res.host(pts, 0)
    d0 = np.sqrt(nb.astype(np.float32)).astype(np.float64)
    d1 = np.where(ns < 0, np.inf, np.sqrt(np.maximum(ns, 0).astype(np.float32)).astype(np.float64))
    i1 = np.where(ns < 0, -1, 0)
    return np.stack([d0, d1], 1), np.stack([idx, i1], 1)


def _ratio_filter(dist, idx, ratio, single_cap):
    """matching.py:82-103 on float64 distances."""
    out = []
    for row in range(len(dist)):
        best, second = dist[row]
        if idx[row, 0] < 0:
            continue
        if idx[row, 1] < 0 or not np.isfinite(second):
            if best < single_cap:
                out.append((row, int(idx[row, 0]), float(best), 0.0))
            continue
        r = best / second if second > 0 else 1.0
        if r < ratio:
            out.append((row, int(idx[row, 0]), float(best), float(r)))
    return out


def ranked_2d2d_search(model, graph, image_id, image_fs, feature_store, *, top_k=RANKED_TOP_K,
                       ratio=RATIO_UNGUIDED, single_cap=SINGLE_CANDIDATE_CAP,
                       min_correspondences=MIN_CORRESPONDENCES, index=None, stats=None):
    """Drop-in for localize.py:125-176 (u8 proxy queries through the device kNN)."""
    from .types import InsufficientDataError

    neighbors = [(graph.match_count(image_id, o), -o, o) for o in graph.neighbors(image_id)
                 if model.is_registered(o)]
    if not neighbors:
        raise InsufficientDataError(f"image {image_id} has no localized neighbours")
    neighbors.sort(reverse=True)
    bank = FeatureBank({int(image_id): image_fs})
    best: dict = {}
    for _, _, other in neighbors[:top_k]:
        proxy = [(pid, model.points[pid].track[other]) for pid in sorted(model.points_visible_in(other))]
        if not proxy:
            continue
        qd = np.stack([feature_store.descriptor(other, f) for _, f in proxy])
        if stats is not None:
            stats.add(len(proxy), len(proxy) * len(image_fs))
        dist, idx = _knn_u8(bank, int(image_id), qd)
        for row, feat, d, _ in _ratio_filter(dist, idx, ratio, single_cap):
            pid = proxy[row][0]
            cur = best.get(pid)
            if cur is None or d < cur[0]:
                best[pid] = (d, feat)
    by_feature: dict = {}
    for pid, (d, feat) in best.items():
        cur = by_feature.get(feat)
        if cur is None or d < cur[0]:
            by_feature[feat] = (d, pid)
    corr = sorted((pid, feat) for feat, (d, pid) in by_feature.items())
    if len(corr) <= min_correspondences:
        return []
    return corr


def _camera(K, R, t, image_id):
    try:  # the caller's own Camera class when running inside msfm
        from msfm.model import Camera as RefCamera  # noqa: F401
        return RefCamera(K=K, R=R, t=t, image_id=image_id)
    except Exception:
        from .types import Camera
        return Camera(K=K, R=R, t=t, image_id=image_id)


def _ref(image_id, fid):
    try:
        from msfm.model import FeatureRef as RefFR
        return RefFR(image_id, fid)
    except Exception:
        from .types import FeatureRef
        return FeatureRef(image_id, fid)


def localize_images(model, graph, image_ids, feature_store, intrinsics, *, cover_points=None,
                    ratio=RATIO_UNGUIDED, min_correspondences=MIN_CORRESPONDENCES,
                    pnp_threshold=4.0, pnp_min_inliers=16, seed=0, stats=None):
    """localize_image (localize.py:179-222) for many images in one device pass.
    Raises OverflowError where the reference's pnp_ransac does."""
    from .pnp import pnp_batch
    from .types import InsufficientDataError

    image_ids = [int(i) for i in image_ids]
    points = cover_points if cover_points is not None else sorted(model.points)
    pts = model_points(model, feature_store, points)
    bank = FeatureBank({i: feature_store.sets[i] for i in image_ids})
    if stats is not None:
        for i in image_ids:
            stats.add(len(points), len(points) * len(feature_store.sets[i]))
    corrs = direct_search(bank, pts, image_ids, ratio=ratio) if len(points) else \
        [np.zeros((0, 2), np.int64) for _ in image_ids]
    methods, corr_lists = {}, {}
    for i, c in zip(image_ids, corrs):
        corr = [(int(p), int(f)) for p, f in c]
        methods[i] = "direct3d2d"
        if len(corr) <= min_correspondences:
            try:
                corr = ranked_2d2d_search(model, graph, i, feature_store.sets[i], feature_store,
                                          ratio=ratio, min_correspondences=min_correspondences,
                                          stats=stats)
            except InsufficientDataError:
                corr = []
            methods[i] = "ranked2d2d"
        corr_lists[i] = corr
    todo = [i for i in image_ids if len(corr_lists[i]) > min_correspondences]
    # positions of every point once, then vectorized gathers per image
    pids_all = np.asarray(sorted({p for i in todo for p, _ in corr_lists[i]}), np.int64)
    pos_all = np.stack([model.points[int(p)].position for p in pids_all]) if len(pids_all) \
        else np.zeros((0, 3))
    X, uv = [], []
    for i in todo:
        c = np.asarray(corr_lists[i], np.int64).reshape(-1, 2)
        X.append(pos_all[np.searchsorted(pids_all, c[:, 0])])
        uv.append(np.asarray(feature_store.sets[i].xy)[c[:, 1]].astype(np.float64))
    res = pnp_batch(X, uv, [intrinsics[i] for i in todo], [seed + i for i in todo],
                    threshold=pnp_threshold, min_inliers=pnp_min_inliers) if todo else []
    pnp = dict(zip(todo, res))
    out = []
    for i in image_ids:
        corr = corr_lists[i]
        if i not in pnp:
            out.append(LocalizationResult(image_id=i, method=methods[i],
                                          reason="below correspondence gate"))
            continue
        r = pnp[i]
        if r.status == "overflow":
            raise OverflowError("cannot convert float infinity to integer")
        if r.status != "ok":
            out.append(LocalizationResult(image_id=i, method=methods[i], correspondences=corr,
                                          reason="resection failed"))
            continue
        pose = _camera(intrinsics[i], r.R, r.t, i)
        refs = [(corr[k][0], _ref(i, corr[k][1])) for k in range(len(corr)) if r.mask[k]]
        out.append(LocalizationResult(image_id=i, method=methods[i], correspondences=corr,
                                      pose=pose, inliers=int(r.mask.sum()), inlier_refs=refs))
    return out


def localize_image(model, graph, image_id, feature_store, intrinsics, *, cover_points=None,
                   ratio=RATIO_UNGUIDED, min_correspondences=MIN_CORRESPONDENCES,
                   pnp_threshold=4.0, pnp_min_inliers=16, seed=0, stats=None):
    """Drop-in for localize.py:179-222."""
    return localize_images(model, graph, [image_id], feature_store, {image_id: intrinsics},
                           cover_points=cover_points, ratio=ratio,
                           min_correspondences=min_correspondences, pnp_threshold=pnp_threshold,
                           pnp_min_inliers=pnp_min_inliers, seed=seed, stats=stats)[0]


def localize_all(model, feature_store, graph, intrinsics, *, iteration=1, set_cover_k=SET_COVER_K,
                 set_cover_engage=SET_COVER_ENGAGE_POINTS, force_set_cover=False,
                 ratio=RATIO_UNGUIDED, min_correspondences=MIN_CORRESPONDENCES,
                 pnp_threshold=4.0, pnp_min_inliers=16, seed=0, threads=1, order=None):
    """Drop-in for localize.py:225-281: one batched device pass over every
    unregistered image, then the image-id-ordered merge."""
    unregistered = [i for i in sorted(feature_store.sets) if not model.is_registered(i)]
    if order is not None:
        wanted = set(unregistered)
        unregistered = [i for i in order if i in wanted]
    if not unregistered:
        model.stage_tag = f"after_localize({iteration})"
        return [], []
    cover = None
    if force_set_cover or len(model.points) > set_cover_engage:
        cover = compute_set_cover(model, set_cover_k).selected
    results = localize_images(model, graph, unregistered, feature_store, intrinsics,
                              cover_points=cover, ratio=ratio,
                              min_correspondences=min_correspondences, pnp_threshold=pnp_threshold,
                              pnp_min_inliers=pnp_min_inliers, seed=seed)
    newly = []
    for r in sorted(results, key=lambda r: r.image_id):
        if r.pose is None:
            continue
        model.attach_camera(r.pose, r.inlier_refs)
        newly.append(r.image_id)
    model.stage_tag = f"after_localize({iteration})"
    return newly, results
