"""Coarse unguided matching on the device: ``match_pair``, ``hybrid_match`` and
``build_coarse_matchgraph`` (matching.py:116-249) over the tcgen05 kNN kernel,
with the pair geometry from the batched device ``estimate_fundamental_ransac``.

The kNN is the reference's exact index (two_nearest_bruteforce,
descriptors.py:35-72; DescriptorIndex takes that path up to 6,400 target
features).  Per query image one kernel launch covers every target image: the
query tier descriptors are the "points" (track length 1) and the targets'
coarse tiers the feature sets.  Distances are the reference's f32 values (exact
integers, sqrt in f32), so ratio test, single-candidate cap and target dedupe
reproduce matching.py:82-113 exactly; hybrid_match's batch / continue /
early-stop schedule (matching.py:143-187) is replayed on the per-row results.
"""

from __future__ import annotations

import numpy as np

from .bank import FeatureBank
from .fundamental import fransac_batch
from .localize import PointSet, knn2_tracks
from .types import Edge, FeatureRef, Match, MatchGraph, TwoViewGeometry

RATIO_UNGUIDED = 0.6            # matching.py:21
SINGLE_CANDIDATE_CAP = 45.0     # matching.py:27
HYBRID_BATCH_FRACTION = 0.10    # matching.py:29
HYBRID_CONTINUE_MIN = 4
HYBRID_EARLY_STOP = 64
MIN_EDGE_MATCHES = 16
MIN_EDGE_INLIERS = 16           # geometry.py:22
PREEMPTIVE_TOP = 100
PREEMPTIVE_MIN_MATCHES = 4
EXACT_LIMIT = 6400              # DescriptorIndex exact path: n <= 32 * 200


def _ref_types():
    try:
        from msfm.geometry import TwoViewGeometry as G
        from msfm.matching import Edge as E, Match as M, MatchGraph as MG
        from msfm.model import FeatureRef as FR
        return FR, M, E, MG, G
    except Exception:
        return FeatureRef, Match, Edge, MatchGraph, TwoViewGeometry


def _knn_rows(bank, qdesc, targets, counts):
    """(idx, d0, d1) per target slot for the u8 query rows: f64 of the f32 sqrt
    distances, d1 = inf without a second neighbour (descriptors.py:35-72)."""
    q = np.asarray(qdesc, dtype=np.int32).reshape(-1, 128)
    pts = PointSet(S=q, n=np.ones(len(q), np.int32), ids=np.arange(len(q)))
    res = knn2_tracks(bank, pts, targets, counts=counts)
    idx, nb, ns = res.host_all(pts)
    d0 = np.sqrt(nb.astype(np.float32)).astype(np.float64)
    d1 = np.where(ns < 0, np.inf, np.sqrt(np.maximum(ns, 0).astype(np.float32)).astype(np.float64))
    return idx, d0, d1


def _ratio_filter(idx, d0, d1, ratio, single_cap):
    """matching.py:82-103 vectorized: (rows, targets, dist, ratio) accepted."""
    has = idx >= 0
    single = ~np.isfinite(d1)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(d1 > 0, d0 / np.where(d1 > 0, d1, 1.0), 1.0)
    acc = has & np.where(single, d0 < single_cap, r < ratio)
    rows = np.flatnonzero(acc)
    return rows, idx[rows], d0[rows], np.where(single[rows], 0.0, r[rows])


def _dedupe(rows, tgts, d, r):
    """matching.py:106-113: one row per target (smaller distance, then row), by row."""
    if len(rows) == 0:
        return rows, tgts, d, r
    order = np.lexsort((rows, d, tgts))
    first = np.ones(len(order), bool)
    first[1:] = tgts[order][1:] != tgts[order][:-1]
    keep = order[first]
    keep = keep[np.argsort(rows[keep], kind="stable")]
    return rows[keep], tgts[keep], d[keep], r[keep]


def _hybrid(idx, d0, d1, n_query_all, n_tier, ratio, batch_fraction, continue_min,
            early_stop, single_cap, n_target_tier, stats):
    """hybrid_match's batch schedule (matching.py:143-187) on per-row kNN results."""
    batch = max(1, int(np.ceil(batch_fraction * n_query_all)))
    rows, tg, dd, rr = _ratio_filter(idx, d0, d1, ratio, single_cap)
    accepted = 0
    end = 0
    first_done = False
    for start in range(0, n_tier, batch):
        if first_done and accepted <= continue_min:
            break
        if accepted >= early_stop:
            break
        stop = min(start + batch, n_tier)
        accepted += int(np.count_nonzero((rows >= start) & (rows < stop)))
        if stats is not None:
            stats.add(stop - start, (stop - start) * n_target_tier)
        end = stop
        first_done = True
    sel = rows < end
    return _dedupe(rows[sel], tg[sel], dd[sel], rr[sel])


def _hybrid_all(idx, d0, d1, n_query_all, n_tier, ratio, batch_fraction, continue_min,
                early_stop, single_cap, n_target_tiers, stats):
    """_hybrid for every target slot of one query image at once (rows = target
    slots of the kNN result): the ratio filter, the batch schedule (accepted counts
    from one cumulative sum) and the per-target dedupe are array operations over
    all slots; returns the per-slot (rows, targets, dist, ratio) in slot order."""
    S = idx.shape[0]
    has = idx >= 0
    single = ~np.isfinite(d1)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(d1 > 0, d0 / np.where(d1 > 0, d1, 1.0), 1.0)
    acc = has & np.where(single, d0 < single_cap, r < ratio)
    batch = max(1, int(np.ceil(batch_fraction * n_query_all)))
    csum = np.cumsum(acc, axis=1)
    accepted = np.zeros(S, np.int64)
    end = np.zeros(S, np.int64)
    active = np.ones(S, bool)
    tiers = np.asarray(n_target_tiers, np.int64)
    first_done = False
    for start in range(0, n_tier, batch):
        if first_done:
            active &= ~(accepted <= continue_min)
        active &= ~(accepted >= early_stop)
        if not active.any():
            break
        stop = min(start + batch, n_tier)
        accepted[active] = csum[active, stop - 1]
        if stats is not None:
            na = int(active.sum())
            stats.add((stop - start) * na, (stop - start) * int(tiers[active].sum()))
        end[active] = stop
        first_done = True
    sel = acc & (np.arange(acc.shape[1])[None, :] < end[:, None])
    ss, rows = np.nonzero(sel)
    tg, dd = idx[ss, rows], d0[ss, rows]
    rr = np.where(single[ss, rows], 0.0, r[ss, rows])
    if len(rows):
        order = np.lexsort((rows, dd, tg, ss))
        first = np.ones(len(order), bool)
        first[1:] = (ss[order][1:] != ss[order][:-1]) | (tg[order][1:] != tg[order][:-1])
        keep = order[first]
        keep = keep[np.lexsort((rows[keep], ss[keep]))]
        ss, rows, tg, dd, rr = ss[keep], rows[keep], tg[keep], dd[keep], rr[keep]
    bnd = np.searchsorted(ss, np.arange(S + 1))
    return [(rows[bnd[s]:bnd[s + 1]], tg[bnd[s]:bnd[s + 1]], dd[bnd[s]:bnd[s + 1]],
             rr[bnd[s]:bnd[s + 1]]) for s in range(S)]


def _matches(types, qid, tid, rows, tgts, d, r, qmap=None, tmap=None):
    FR, M = types[0], types[1]
    qm = rows if qmap is None else qmap[rows]
    tm = tgts if tmap is None else tmap[tgts]
    return [M(query=FR(qid, a), target=FR(tid, b), distance=c, ratio=e)
            for a, b, c, e in zip(np.asarray(qm).tolist(), np.asarray(tm).tolist(),
                                  np.asarray(d, np.float64).tolist(),
                                  np.asarray(r, np.float64).tolist())]


def match_pair(query_fs, target_fs, *, ratio=RATIO_UNGUIDED, query_indices=None,
               target_indices=None, single_cap=SINGLE_CANDIDATE_CAP, index=None, stats=None):
    """Drop-in for msfm.matching.match_pair (matching.py:116-140), exact index."""
    types = _ref_types()
    qi = np.arange(query_fs.coarse_count) if query_indices is None else np.asarray(query_indices)
    ti = np.arange(target_fs.coarse_count) if target_indices is None else np.asarray(target_indices)
    if len(qi) == 0 or len(ti) == 0:
        return []
    sub = _Sub(target_fs, ti)
    bank = FeatureBank({0: sub})
    idx, d0, d1 = _knn_rows(bank, np.asarray(query_fs.descriptors)[qi], [0], None)
    if stats is not None:
        stats.add(len(qi), len(qi) * len(ti))
    rows, tg, dd, rr = _dedupe(*_ratio_filter(idx[0], d0[0], d1[0], ratio, single_cap))
    return _matches(types, query_fs.image_id, target_fs.image_id, rows, tg, dd, rr, qi, ti)


def hybrid_match(query_fs, target_fs, *, ratio=RATIO_UNGUIDED,
                 batch_fraction=HYBRID_BATCH_FRACTION, continue_min=HYBRID_CONTINUE_MIN,
                 early_stop=HYBRID_EARLY_STOP, single_cap=SINGLE_CANDIDATE_CAP, stats=None):
    """Drop-in for msfm.matching.hybrid_match (matching.py:143-187)."""
    types = _ref_types()
    n_tier, m_tier = int(query_fs.coarse_count), int(target_fs.coarse_count)
    if n_tier == 0 or m_tier == 0:
        return []
    bank = FeatureBank({0: target_fs})
    idx, d0, d1 = _knn_rows(bank, np.asarray(query_fs.descriptors)[:n_tier], [0],
                            np.array([m_tier]))
    rows, tg, dd, rr = _hybrid(idx[0], d0[0], d1[0], len(query_fs), n_tier, ratio, batch_fraction,
                               continue_min, early_stop, single_cap, m_tier, stats)
    return _matches(types, query_fs.image_id, target_fs.image_id, rows, tg, dd, rr)


class _Sub:
    """Row subset of a FeatureSet with the attributes the bank reads."""

    def __init__(self, fs, idx):
        self.xy = np.asarray(fs.xy)[idx]
        self.descriptors = np.asarray(fs.descriptors)[idx]
        self.width, self.height = fs.width, fs.height

    def __len__(self):
        return len(self.xy)


def preemptive_pair_filter(feature_sets, *, n_top=PREEMPTIVE_TOP,
                           min_matches=PREEMPTIVE_MIN_MATCHES, ratio=RATIO_UNGUIDED):
    """Drop-in for matching.py:190-205: match_pair over each image's top features."""
    ids = sorted(feature_sets)
    bank = FeatureBank({i: feature_sets[i] for i in ids})
    tops = np.array([min(n_top, len(feature_sets[i])) for i in ids], np.int64)
    kept = []
    for ai, a in enumerate(ids[:-1]):
        targets = ids[ai + 1:]
        if tops[ai] == 0:
            continue
        idx, d0, d1 = _knn_rows(bank, np.asarray(feature_sets[a].descriptors)[:tops[ai]],
                                targets, tops)
        for s, b in enumerate(targets):
            if tops[ai + 1 + s] == 0:
                continue
            rows, *_ = _dedupe(*_ratio_filter(idx[s], d0[s], d1[s], ratio, SINGLE_CANDIDATE_CAP))
            if len(rows) >= min_matches:
                kept.append((a, b))
    return kept


def build_coarse_matchgraph(feature_sets, *, ratio=RATIO_UNGUIDED, preemptive=False,
                            min_edge_matches=MIN_EDGE_MATCHES, min_edge_inliers=MIN_EDGE_INLIERS,
                            early_stop=HYBRID_EARLY_STOP, seed=0, threads=1, stats=None,
                            on_overflow="raise"):
    """Drop-in for msfm.matching.build_coarse_matchgraph (matching.py:208-249):
    one kNN launch per query image over all its candidate partners, the hybrid
    schedule per pair, then one batched device RANSAC over every surviving pair.

    A pair whose RANSAC hits the reference's OverflowError (geometry.py:189, a
    best inlier fraction below ~1%) raises it, as the reference does;
    ``on_overflow="drop"`` (not the reference's behaviour) drops such pairs and
    counts them in ``graph.overflow_pairs`` instead."""
    FR, M, E, MG, G = _ref_types()
    ids = sorted(feature_sets)
    if preemptive:
        pairs = preemptive_pair_filter(feature_sets, ratio=ratio)
    else:
        pairs = [(a, b) for i, a in enumerate(ids) for b in ids[i + 1:]]
    partners = {}
    for a, b in pairs:
        partners.setdefault(a, []).append(b)
    bank = FeatureBank({i: feature_sets[i] for i in ids})
    tiers = np.array([int(feature_sets[i].coarse_count) for i in ids], np.int64)
    pos = {i: k for k, i in enumerate(ids)}
    hybrid = {}
    for a in sorted(partners):
        fa = feature_sets[a]
        n_tier = int(fa.coarse_count)
        targets = [b for b in partners[a] if tiers[pos[b]] > 0]
        for b in partners[a]:
            hybrid[(a, b)] = None
        if n_tier == 0 or not targets:
            continue
        idx, d0, d1 = _knn_rows(bank, np.asarray(fa.descriptors)[:n_tier], targets, tiers)
        per = _hybrid_all(idx, d0, d1, len(fa), n_tier, ratio, HYBRID_BATCH_FRACTION,
                          HYBRID_CONTINUE_MIN, early_stop, SINGLE_CANDIDATE_CAP,
                          [int(tiers[pos[b]]) for b in targets], stats)
        for b, h in zip(targets, per):
            hybrid[(a, b)] = h
    cand, q_list, c_list, seeds = [], [], [], []
    xy64 = {}

    def xy_of(i):
        v = xy64.get(i)
        if v is None:
            v = xy64[i] = np.asarray(feature_sets[i].xy, np.float64)
        return v

    for a, b in pairs:
        h = hybrid.get((a, b))
        if h is None or len(h[0]) < min_edge_matches:
            continue
        rows, tg = h[0], h[1]
        cand.append((a, b))
        q_list.append(xy_of(a)[rows])
        c_list.append(xy_of(b)[tg])
        seeds.append(seed + a * 100003 + b)
    geo = fransac_batch(q_list, c_list, seeds) if cand else []
    graph = MG()
    dropped = []
    for (a, b), g in zip(cand, geo):
        if g.status == "overflow":
            if on_overflow == "drop":
                dropped.append((a, b))
                continue
            raise OverflowError("cannot convert float infinity to integer")   # geometry.py:189
        if int(g.mask.sum()) < min_edge_inliers:
            continue
        rows, tg, dd, rr = hybrid[(a, b)]
        # Python scalars first (.tolist()): the objects are built without numpy scalars
        ms = [M(query=FR(a, x), target=FR(b, y), distance=c, ratio=e)
              for x, y, c, e in zip(rows.tolist(), tg.tolist(), dd.tolist(), rr.tolist())]
        geom = G(F=g.F, inlier_count=g.inlier_count, degenerate_planar=g.degenerate_planar)
        graph.edges[(a, b)] = E(matches=ms, geometry=geom, inlier_mask=g.mask)
    if on_overflow == "drop":
        graph.overflow_pairs = dropped
    return graph
