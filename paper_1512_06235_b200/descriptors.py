"""Drop-ins for ``msfm.descriptors`` (descriptors.py:23-139) on the tcgen05 kNN.

``two_nearest_bruteforce`` and ``DescriptorIndex.knn2`` return the reference's
(dist, idx) arrays: top-2 by squared L2 with the lowest index winning ties,
distances ``sqrt`` of the f32 value as float64, second column +inf / -1 when the
target set has a single row.  The device computes integer distances exactly, which
equals the reference's f32 arithmetic whenever the queries are integer-valued
(uint8 descriptors: every partial sum stays below 2^24) — the case of match_pair,
hybrid_match and ranked_2d2d_search.  Rows that are not integer-valued in
[0, 255] (arbitrary float32 input) go to ``msfm_knn2_float``: the squared
distance summed in f64 from exact f32 differences, lowest index on ties — the
real-valued answer the reference's f32 ``|q|^2 + |t|^2 - 2 q.t`` approximates
(the two can order near-ties differently; distances are the f64 value's sqrt).
The 3D-2D search itself uses the exact (S, n) track-sum form
(localize.direct_search).  The reference switches to an approximate kd-tree above
``leaf_size * max_leaf_visits`` targets; this index always answers exactly, and
``DescriptorIndex.exact`` reports the reference's own choice of path.
"""

from __future__ import annotations

import numpy as np

from .bank import FeatureBank
from .localize import PointSet, knn2_tracks
from .types import SearchStats

EXACT_THRESHOLD = 2000     # descriptors.py:16
LEAF_SIZE = 32
MAX_LEAF_VISITS = 200


class _Rows:
    def __init__(self, desc):
        n = len(desc)
        self.descriptors = desc
        self.xy = np.zeros((n, 2), np.float32)
        self.width, self.height = 1, 1

    def __len__(self):
        return len(self.descriptors)


def _as_u8(a):
    """uint8 rows when ``a`` is integer-valued in [0, 255] with 128 columns, else None."""
    a = np.asarray(a)
    if a.ndim != 2 or a.shape[1] != 128:
        return None
    if a.size == 0:
        return np.zeros((0, 128), np.uint8)
    f = a.astype(np.float64)
    if not (np.all(f == np.round(f)) and f.min() >= 0 and f.max() <= 255):
        return None
    return np.ascontiguousarray(f.astype(np.uint8))


def _knn2_float(targets, queries):
    """Real-valued top-2 on the device (msfm_knn2_float)."""
    import torch

    from . import _lib

    q = np.ascontiguousarray(queries, dtype=np.float32)
    t = np.ascontiguousarray(targets, dtype=np.float32)
    nq, nt = len(q), len(t)
    dist = np.full((nq, 2), np.inf)
    idx = np.full((nq, 2), -1, dtype=np.int64)
    if nq == 0 or nt == 0:
        return dist, idx
    if q.ndim != 2 or t.ndim != 2 or q.shape[1] != t.shape[1]:
        raise ValueError(f"descriptor widths differ: {q.shape} vs {t.shape}")
    lib = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    dq = torch.from_numpy(q).to(dev)
    dt = torch.from_numpy(t).to(dev)
    d2 = torch.empty((nq, 2), dtype=torch.float64, device=dev)
    di = torch.empty((nq, 2), dtype=torch.int64, device=dev)
    _lib.check(lib.msfm_knn2_float(dq.data_ptr(), nq, dt.data_ptr(), nt, q.shape[1],
                                   d2.data_ptr(), di.data_ptr(), _lib.stream_handle()),
               "msfm_knn2_float")
    d2h, dih = d2.cpu().numpy(), di.cpu().numpy()
    dist[:, 0] = np.sqrt(d2h[:, 0])
    idx[:, 0] = dih[:, 0]
    if nt > 1:
        dist[:, 1] = np.sqrt(d2h[:, 1])
        idx[:, 1] = dih[:, 1]
    return dist, idx


def _knn2(targets_u8, queries_u8, bank=None):
    nq, nt = len(queries_u8), len(targets_u8)
    dist = np.full((nq, 2), np.inf)
    idx = np.full((nq, 2), -1, dtype=np.int64)
    if nq == 0 or nt == 0:
        return dist, idx
    bank = bank if bank is not None else FeatureBank({0: _Rows(targets_u8)})
    pts = PointSet(S=queries_u8.astype(np.int32), n=np.ones(nq, np.int32), ids=np.arange(nq))
    # the second neighbour's index (the lowest-index row at the second distance other
    # than the best, descriptors.py:61-63) is resolved by a second device pass
    res = knn2_tracks(bank, pts, [0], second=True)
    i1, nb, ns = res.host(pts, 0)
    i2 = res.i2[0, :nq].cpu().numpy().astype(np.int64)
    dist[:, 0] = np.sqrt(nb.astype(np.float32)).astype(np.float64)
    idx[:, 0] = i1
    if nt > 1:
        dist[:, 1] = np.sqrt(ns.astype(np.float32)).astype(np.float64)
        idx[:, 1] = i2
    return dist, idx


def two_nearest_bruteforce(queries, targets, stats: SearchStats | None = None):
    """Drop-in for msfm.descriptors.two_nearest_bruteforce (descriptors.py:35-72)."""
    q, t = _as_u8(queries), _as_u8(targets)
    if stats is not None:
        stats.add(len(queries), len(queries) * len(targets))
    if q is None or t is None:
        return _knn2_float(targets, queries)
    return _knn2(t, q)


class DescriptorIndex:
    """Drop-in for msfm.descriptors.DescriptorIndex (descriptors.py:105-139): the
    target rows live on the device; every query is answered exactly."""

    def __init__(self, descriptors, *, exact_threshold: int = EXACT_THRESHOLD,
                 leaf_size: int = LEAF_SIZE, max_leaf_visits: int = MAX_LEAF_VISITS):
        self.data = np.ascontiguousarray(descriptors, dtype=np.float32)
        self.n = len(self.data)
        self.leaf_size = leaf_size
        self.max_leaf_visits = max_leaf_visits
        # the reference's choice of path (descriptors.py:117-119); answers here are
        # exact either way
        self.exact = self.n <= exact_threshold or self.n <= leaf_size * max_leaf_visits
        self._u8 = _as_u8(self.data)
        self._bank = FeatureBank({0: _Rows(self._u8)}) if self.n and self._u8 is not None else None

    def knn2(self, queries, stats: SearchStats | None = None):
        q = _as_u8(queries)
        if stats is not None:
            stats.add(len(queries), len(queries) * self.n)
        if q is None or self._u8 is None:
            return _knn2_float(self.data, queries)
        return _knn2(self._u8, q, self._bank)
