"""Point addition stage (densify.py:168-286 of the reference) over the device path.

Pairs come from covisibility (a sparse V·Vᵀ instead of per-pair set
intersections), all pairs are matched in one batched ``match_pairs`` call,
tracks are merged on the host (``merge_tracks``: the reference's connected
components and conflict rules, densify.py:68-158, over integer feature keys
with union-find), and all new / grown tracks are triangulated in one batched
kernel launch.  The model is then updated in the reference's order.
"""

from __future__ import annotations

import numpy as np

from .bank import FeatureBank
from .geometry import fundamental_from_poses
from .guided import BAND_D_PX, GRID_INFLATION, RATIO_GUIDED, match_pairs
from .triangulation import triangulate_batch
from .types import DegenerateGeometryError, NotRegisteredError

COVIS_THRESHOLD = 8
CANDIDATE_FRACTION = 0.10


def _key(i, f):
    return (int(i) << 32) | int(f)


def _ref_type():
    try:
        from msfm.model import FeatureRef
        return FeatureRef
    except Exception:
        from .types import FeatureRef
        return FeatureRef


def covisibility_counts(model, ids):
    """len(model.covisible_points(a, b)) for all registered pairs (model.py:105-110)."""
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


def candidate_pairs(model, query_images, threshold, k_limit):
    ids = model.image_ids()
    C = covisibility_counts(model, ids)
    pos = {i: k for k, i in enumerate(ids)}
    pairs = set()
    for i in query_images:
        if not model.is_registered(i):
            raise NotRegisteredError(f"image {i} is not registered")
        a = pos[i]
        scored = sorted((-int(C[a, pos[o]]), o) for o in ids if o != i and C[a, pos[o]] > threshold)
        for _, o in scored[:k_limit]:
            pairs.add((i, o) if i < o else (o, i))
    return sorted(pairs)


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


def densify_stage(model, feature_store, *, iteration=1, query_images=None, d=BAND_D_PX,
                  ratio=RATIO_GUIDED, inflation=GRID_INFLATION, threshold=COVIS_THRESHOLD,
                  candidate_fraction=CANDIDATE_FRACTION, tri_max_error_px=4.0,
                  tri_min_angle_deg=1.0, threads=1, stats=None) -> dict:
    """Drop-in for msfm.densify.densify_stage."""
    FR = _ref_type()
    registered = model.image_ids()
    if query_images is None:
        query_images = registered
    query_images = [i for i in sorted(query_images) if model.is_registered(i)]
    k_limit = max(1, int(np.ceil(candidate_fraction * len(registered))))
    pairs = candidate_pairs(model, query_images, threshold, k_limit)
    qset = set(query_images)
    imgs = sorted({x for p in pairs for x in p})
    untracked = {}
    for i in imgs:
        n = len(feature_store.sets[i])
        owned = np.zeros(n, bool)
        for pid in model.points_visible_in(i):
            owned[model.points[pid].track[i]] = True
        untracked[i] = np.flatnonzero(~owned).astype(np.int32)
    q_img, t_img, Fs, ok = [], [], [], []
    for a, b in pairs:
        q, t = (a, b) if a in qset else (b, a)
        try:
            F = fundamental_from_poses(model.cameras[q], model.cameras[t]).F
        except DegenerateGeometryError:
            F = None
        q_img.append(q)
        t_img.append(t)
        Fs.append(F if F is not None else np.full((3, 3), np.nan))
        ok.append(F is not None)
    all_q, all_qf, all_t, all_tf, all_d = [], [], [], [], []
    if pairs:
        bank = FeatureBank({i: feature_store.sets[i] for i in imgs})
        res = match_pairs(bank, q_img, t_img, np.stack(Fs), [untracked[q] for q in q_img], d=d,
                          ratio=ratio, inflation=inflation, with_stats=stats is not None)
        pk, mq, mt, md, _ = res.to_host()
        if stats is not None:
            s = res.stats.cpu().numpy()
            stats.add(int(s[:, 0].sum()), int(s[:, 1].sum()))
        qa, ta = np.asarray(q_img), np.asarray(t_img)
        all_q, all_qf, all_t, all_tf, all_d = qa[pk], mq, ta[pk], mt, md.astype(np.float64)
    n_matches = len(all_q)
    new_tracks, extensions = merge_tracks(all_q, all_qf, all_t, all_tf, all_d, model)
    # grown tracks: reference order, fresh refs against the current ownership
    ext_jobs = []
    for pid in sorted(extensions):
        fresh = [k for k in sorted(set(extensions[pid]))
                 if model.owner(FR(k >> 32, k & 0xFFFFFFFF)) is None
                 and (k >> 32) not in model.points[pid].track]
        if fresh:
            cand = [_key(r.image_id, r.feature_id) for r in model.points[pid].refs()] + fresh
            ext_jobs.append((pid, fresh, cand))
    tracks = [t for t in new_tracks] + [c for _, _, c in ext_jobs]
    cams = sorted(model.cameras)
    cpos = {c: k for k, c in enumerate(cams)}
    K = np.stack([model.cameras[c].K for c in cams]) if cams else np.zeros((0, 3, 3))
    R = np.stack([model.cameras[c].R for c in cams]) if cams else np.zeros((0, 3, 3))
    t = np.stack([model.cameras[c].t for c in cams]) if cams else np.zeros((0, 3))
    ptr = np.zeros(len(tracks) + 1, np.int64)
    np.cumsum([len(x) for x in tracks], out=ptr[1:])
    flat = [k for x in tracks for k in x]
    cam = np.array([cpos[k >> 32] for k in flat], np.int32)
    pix = np.array([feature_store.position(k >> 32, k & 0xFFFFFFFF) for k in flat],
                   np.float64).reshape(-1, 2)
    if tracks:
        st, X, _ = triangulate_batch(K, R, t, ptr, cam, pix, max_error=tri_max_error_px,
                                     min_angle_deg=tri_min_angle_deg)
    else:
        st, X = np.zeros(0, np.int32), np.zeros((0, 3))
    added = extended = 0
    for j, refs in enumerate(new_tracks):
        if st[j] == -1:
            raise DegenerateGeometryError("triangulation rays are parallel or share one centre")
        if st[j] != 1:
            continue
        model.add_point(X[j], [FR(k >> 32, k & 0xFFFFFFFF) for k in refs])
        added += 1
    base = len(new_tracks)
    for j, (pid, fresh, _) in enumerate(ext_jobs):
        s = st[base + j]
        if s == -1:
            raise DegenerateGeometryError("triangulation rays are parallel or share one centre")
        if s != 1:
            continue
        for k in fresh:
            model.extend_track(pid, FR(k >> 32, k & 0xFFFFFFFF))
        model.set_position(pid, X[base + j])
        extended += 1
    model.stage_tag = f"after_densify({iteration})"
    return {"pairs": len(pairs), "matches": n_matches, "new_points": added,
            "extended_tracks": extended}
