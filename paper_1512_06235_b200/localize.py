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

RATIO_UNGUIDED = 0.6     # matching.py:21
SINGLE_CANDIDATE_CAP = 45.0
MIN_CORRESPONDENCES = 16  # localize.py:30
INT_BIG = 0x7FFFFFFF


def ratio_fraction(ratio: float):
    f = Fraction(float(ratio)).limit_denominator(1 << 20)
    return f.numerator, f.denominator


@dataclass
class PointSet:
    """Exact query points: track sums S (M,128) int32, lengths n (M,), ids."""

    S: np.ndarray
    n: np.ndarray
    ids: np.ndarray

    @property
    def SS(self) -> np.ndarray:
        S = self.S.astype(np.int64)
        return (S * S).sum(1)


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

    def host(self, pts: PointSet, s: int):
        """(idx, N_best, N_second) of query slot s, N_second=-1 if undefined."""
        M = len(pts.n)
        k1 = self.k1[s, :M].cpu().numpy().astype(np.int64)
        i1 = self.i1[s, :M].cpu().numpy().astype(np.int64)
        k2 = self.k2[s, :M].cpu().numpy().astype(np.int64)
        n = pts.n.astype(np.int64)
        SS = pts.SS
        Nb = n * k1 + SS
        Ns = np.where(k2 == INT_BIG, -1, n * k2 + SS)
        return i1, Nb, Ns


def knn2_tracks(bank: FeatureBank, pts: PointSet, image_ids, stream=None,
                device_points=None) -> DeviceKnn:
    import torch

    lib = _lib.load()
    M = len(pts.n)
    M_pad = (M + 127) // 128 * 128
    dev = bank.device
    if device_points is None:
        device_points = upload_points(pts, dev)
    dS, dn, dSS = device_points
    slots = np.array([bank.index_of[int(i)] for i in image_ids], dtype=np.int32)
    d_slots = torch.from_numpy(slots).to(dev)
    k1 = torch.empty((max(len(slots), 1), M_pad), dtype=torch.int32, device=dev)
    i1 = torch.empty_like(k1)
    k2 = torch.empty_like(k1)
    ws_bytes = lib.msfm_knn_workspace_bytes(M)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    b = bank.cstruct()
    maxn = int(pts.n.max()) if M else 0
    _lib.check(lib.msfm_knn2_tracks(ctypes.byref(b), M, _lib.ptr(dS), _lib.ptr(dn), len(slots),
                                    _lib.ptr(d_slots), maxn, _lib.ptr(k1), _lib.ptr(i1),
                                    _lib.ptr(k2), _lib.ptr(ws), ws_bytes,
                                    _lib.stream_handle(stream)), "msfm_knn2_tracks")
    return DeviceKnn(k1, i1, k2, M_pad, keep=(ws, d_slots))


def upload_points(pts: PointSet, dev):
    import torch

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)

    M = len(pts.n)
    return (up(pts.S.astype(np.int32) if M else np.zeros((1, 128), np.int32)),
            up(pts.n.astype(np.int32) if M else np.zeros(1, np.int32)),
            up(pts.SS if M else np.zeros(1, np.int64)))


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
                  knn: DeviceKnn | None = None, to_host: bool = True):
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
    d_slots = torch.from_numpy(slots).to(dev)
    nfeat = bank.counts[slots].astype(np.int64)
    win_off = np.zeros(len(slots), np.int64)
    if len(slots) > 1:
        np.cumsum(nfeat[:-1], out=win_off[1:])
    d_win_off = torch.from_numpy(win_off).to(dev)
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
    if to_host:
        c = cnt.cpu().numpy()
        return [np.stack([pts.ids[rows[s, :c[s]].cpu().numpy()], fids[s, :c[s]].cpu().numpy()], 1)
                .astype(np.int64) for s in range(len(slots))]
    return res
