"""CPU restatement of the densification track merge (densify.py:68-158).

TEST INFRASTRUCTURE: only tests/ use it, as the checker of the device merge
(``paper_1512_06235_b200.densify.merge_tracks_device``); nothing in the package
imports it.  Parity: the densify fixtures (tests/golden/densify_*.npz) pin the
whole stage against the reference.
"""

from __future__ import annotations

import numpy as np


def _key(i, f):
    return (int(i) << 32) | int(f)


def _ref_type():
    try:
        from msfm.model import FeatureRef
        return FeatureRef
    except Exception:
        from paper_1512_06235_b200.types import FeatureRef
        return FeatureRef


def merge_tracks(q_img, q_fid, t_img, t_fid, dist, model):
    """Connected components over feature keys seeded with the touched model
    tracks, conflict rules of densify.py:121-157.  Returns (new_tracks,
    extensions) as lists of (image, fid) tuples, in the reference's order."""
    nodes = {}
    parent = []

    def node(k):
        j = nodes.get(k)
        if j is None:
            j = len(parent)
            nodes[k] = j
            parent.append(j)
        return j

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    def union(a, b):
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[max(ra, rb)] = min(ra, rb)

    edge = {}
    adj = {}
    for qi, qf, ti, tf, d in zip(q_img, q_fid, t_img, t_fid, dist):
        u, v = _key(qi, qf), _key(ti, tf)
        a, b = node(u), node(v)
        union(a, b)
        e = (u, v) if u < v else (v, u)
        cur = edge.get(e)
        if cur is None or d < cur:
            edge[e] = float(d)
        adj.setdefault(u, []).append(v)
        adj.setdefault(v, []).append(u)
    FR = _ref_type()
    owner_of = {}
    touched = set()
    for k in list(nodes):
        pid = model.owner(FR(k >> 32, k & 0xFFFFFFFF))
        if pid is not None:
            owner_of[k] = pid
            touched.add(pid)
    existing = {}
    for pid in touched:
        refs = [_key(r.image_id, r.feature_id) for r in model.points[pid].refs()]
        existing[pid] = set(refs)
        for k in refs:
            owner_of[k] = pid
            node(k)
        for k in refs[1:]:
            union(nodes[refs[0]], nodes[k])
    comps = {}
    for k, j in nodes.items():
        comps.setdefault(find(j), []).append(k)
    new_tracks, extensions = [], {}
    for comp in sorted(comps.values(), key=min):
        comp.sort()
        owners = {owner_of[k] for k in comp if k in owner_of}
        if len(owners) >= 2:
            continue        # bridges two points: ambiguous, dropped
        owner = owners.pop() if owners else None
        ex = existing.get(owner, set())

        def support(k):
            ds = [edge[(min(k, o), max(k, o))] for o in adj.get(k, ())]
            return min(ds) if ds else np.inf

        by_image = {}
        for k in comp:
            by_image.setdefault(k >> 32, []).append(k)
        keep = []
        for img in sorted(by_image):
            ks = by_image[img]
            pinned = [k for k in ks if k in ex]
            if pinned:
                keep.extend(pinned)
                continue
            if owner is not None and img in model.points[owner].track:
                continue
            ks.sort(key=lambda k: (support(k), k))
            keep.append(ks[0])
        fresh = [k for k in keep if k not in ex]
        if owner is not None:
            if fresh:
                extensions.setdefault(owner, []).extend(fresh)
        elif len(fresh) >= 2 and len({k >> 32 for k in fresh}) >= 2:
            new_tracks.append(fresh)
    return new_tracks, extensions




def covisibility_counts(model, ids):
    """Host restatement (checker): len(model.covisible_points(a, b)), model.py:105-110."""
    pos = {i: k for k, i in enumerate(ids)}
    rows, cols = [], []
    for pid, pt in model.points.items():
        for i in pt.track:
            if i in pos:
                rows.append(pos[i])
                cols.append(pid)
    if not rows:
        return np.zeros((len(ids), len(ids)), np.int64)
    pids = np.unique(cols)
    V = np.zeros((len(ids), len(pids)), np.float32)
    V[np.array(rows), np.searchsorted(pids, np.array(cols))] = 1.0
    return (V @ V.T).astype(np.int64)


