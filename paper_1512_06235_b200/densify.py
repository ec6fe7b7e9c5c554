"""Point addition stage (densify.py:168-286 of the reference) over the device path.

Pairs come from covisibility (a sparse V·Vᵀ instead of per-pair set
intersections), all pairs are matched in one batched ``match_pairs`` call,
tracks are merged on the device (``merge_tracks_device``: the reference's
connected components and conflict rules, densify.py:68-158, as a lock-free
union-find over bank feature rows), and all new / grown tracks are triangulated
in one batched kernel launch.  The model is then updated in the reference's order.
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


def covisibility_counts(model, ids, device=None):
    """len(model.covisible_points(a, b)) for all registered pairs (model.py:105-110),
    counted on the device (msfm_covisibility): int64 (N, N), N = len(ids)."""
    import torch

    from . import _lib

    lib = _lib.load()
    dev = torch.device(device or "cuda")
    pos = {i: k for k, i in enumerate(ids)}
    ptr = [0]
    img = []
    for pid in sorted(model.points):
        for i in model.points[pid].track:
            k = pos.get(i)
            if k is not None:
                img.append(k)
        ptr.append(len(img))
    N = len(ids)
    d_ptr = torch.tensor(ptr, dtype=torch.int64, device=dev)
    d_img = torch.tensor(img if img else [0], dtype=torch.int32, device=dev)
    C = torch.empty((max(N, 1), max(N, 1)), dtype=torch.int32, device=dev)
    _lib.check(lib.msfm_covisibility(len(ptr) - 1, _lib.ptr(d_ptr), _lib.ptr(d_img), N,
                                     _lib.ptr(C), _lib.stream_handle(None)), "msfm_covisibility")
    return C[:N, :N].cpu().numpy().astype(np.int64)


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


def model_tracks(model, bank):
    """(pids, CSR ptr, bank nodes) of every model point's refs inside the bank."""
    pids = sorted(model.points)
    ptr = np.zeros(len(pids) + 1, np.int64)
    nodes = []
    for r, pid in enumerate(pids):
        for ref in model.points[pid].refs():
            k = bank.index_of.get(int(ref.image_id))
            if k is not None:
                nodes.append(int(bank.offsets[k]) + int(ref.feature_id))
        ptr[r + 1] = len(nodes)
    return pids, ptr, np.asarray(nodes, np.int32)


def merge_tracks_nodes(bank, u, v, dist, track_ptr, track_node, stream=None):
    """msfm_merge_tracks on bank nodes: ``u``, ``v`` (device int32) and ``dist``
    (device f32) are the matches, ``track_ptr`` / ``track_node`` (host CSR) the
    model tracks.  Returns host arrays (nodes, segment owners, segment offsets):
    fresh nodes grouped per component in the reference's order, owner = track row
    being extended or -1 for a new track."""
    import ctypes

    import torch

    from . import _lib

    lib = _lib.load()
    dev = bank.device
    d_ptr = torch.from_numpy(np.ascontiguousarray(track_ptr, np.int64)).to(dev)
    tn = np.ascontiguousarray(track_node, np.int32)
    d_tnode = torch.from_numpy(tn if len(tn) else np.zeros(1, np.int32)).to(dev)
    E = int(u.numel())
    # fresh nodes are distinct bank rows touched by the edges
    cap = max(min(2 * E, int(bank.n_total)), 1)
    out_node = torch.empty(cap, dtype=torch.int32, device=dev)
    seg_owner = torch.empty(cap, dtype=torch.int32, device=dev)
    seg_off = torch.empty(cap + 1, dtype=torch.int64, device=dev)
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    ws_bytes = lib.msfm_merge_workspace_bytes(bank.n_total, E)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    b = bank.cstruct()
    _lib.check(lib.msfm_merge_tracks(ctypes.byref(b), E, _lib.ptr(u), _lib.ptr(v), _lib.ptr(dist),
                                     len(track_ptr) - 1, _lib.ptr(d_ptr), _lib.ptr(d_tnode),
                                     _lib.ptr(out_node), _lib.ptr(seg_owner), _lib.ptr(seg_off),
                                     _lib.ptr(counts), _lib.ptr(ws), ws_bytes,
                                     _lib.stream_handle(stream)), "msfm_merge_tracks")
    nseg, nout = (int(x) for x in counts.cpu().numpy())
    return (out_node[:nout].cpu().numpy().astype(np.int64), seg_owner[:nseg].cpu().numpy(),
            seg_off[:nseg + 1].cpu().numpy())


def merge_tracks_device(bank, u, v, dist, model, stream=None, arrays=None):
    """Track merge on the device (msfm_merge_tracks, densify.py:68-158).

    ``u``, ``v`` are bank node ids (device int32), ``dist`` the f32 match
    distances (device).  Returns (new_tracks, extensions) like the reference:
    lists of (image << 32 | feature) keys in component order.  ``arrays`` (a
    dict, optional) receives the raw (nodes, owners, offsets)."""
    pids, ptr, tnode = model_tracks(model, bank)
    nodes, owners, offs = merge_tracks_nodes(bank, u, v, dist, ptr, tnode, stream)
    if arrays is not None:
        arrays.update(nodes=nodes, owners=owners, offs=offs)
    slot = np.searchsorted(bank.offsets, nodes, side="right") - 1
    ids = np.asarray(bank.image_ids, np.int64)
    keys = ((ids[slot] << 32) | (nodes - bank.offsets[slot])).tolist()
    new_tracks, extensions = [], {}
    for s in range(len(owners)):
        seg = keys[offs[s]:offs[s + 1]]
        if owners[s] < 0:
            new_tracks.append(seg)
        else:
            extensions[pids[owners[s]]] = seg
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
    n_matches = 0
    new_tracks, extensions = [], {}
    merged = {}
    if pairs:
        import torch

        bank = FeatureBank({i: feature_store.sets[i] for i in imgs})
        res = match_pairs(bank, q_img, t_img, np.stack(Fs), [untracked[q] for q in q_img], d=d,
                          ratio=ratio, inflation=inflation, with_stats=stats is not None)
        if stats is not None:
            s = res.stats.cpu().numpy()
            stats.add(int(s[:, 0].sum()), int(s[:, 1].sum()))
        rows, n_matches = res.packed()
        # bank nodes of both ends of every match, on the device
        qoff = torch.from_numpy(np.array([bank.offsets[bank.index_of[q]] for q in q_img],
                                         np.int64)).to(bank.device)
        toff = torch.from_numpy(np.array([bank.offsets[bank.index_of[t]] for t in t_img],
                                         np.int64)).to(bank.device)
        pk = rows[:, 0].long()
        qt = rows[:, 1]
        u = (qoff[pk] + (qt & 0xFFFF).long()).to(torch.int32).contiguous()
        v = (toff[pk] + ((qt >> 16) & 0xFFFF).long()).to(torch.int32).contiguous()
        dist = rows[:, 2].contiguous().view(torch.float32)
        new_tracks, extensions = merge_tracks_device(bank, u, v, dist, model, arrays=merged)
    # grown tracks: reference order, fresh refs against the current ownership
    ext_jobs = []
    for pid in sorted(extensions):
        fresh = [k for k in sorted(set(extensions[pid]))
                 if model.owner(FR(k >> 32, k & 0xFFFFFFFF)) is None
                 and (k >> 32) not in model.points[pid].track]
        if fresh:
            cand = [_key(r.image_id, r.feature_id) for r in model.points[pid].refs()] + fresh
            ext_jobs.append((pid, fresh, cand))
    cams = sorted(model.cameras)
    K = np.stack([model.cameras[c].K for c in cams]) if cams else np.zeros((0, 3, 3))
    R = np.stack([model.cameras[c].R for c in cams]) if cams else np.zeros((0, 3, 3))
    t = np.stack([model.cameras[c].t for c in cams]) if cams else np.zeros((0, 3))
    # triangulation input as arrays: the new tracks straight from the merge's
    # segments (bank rows), then the grown tracks' candidate refs
    n_tr = len(new_tracks) + len(ext_jobs)
    lens = [len(x) for x in new_tracks] + [len(c) for _, _, c in ext_jobs]
    ptr = np.zeros(n_tr + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    if merged:
        nodes, owners, offs = (np.asarray(merged[k]) for k in ("nodes", "owners", "offs"))
        sel = np.flatnonzero(owners < 0)
        new_rows = (np.concatenate([nodes[offs[s]:offs[s + 1]] for s in sel]).astype(np.int64)
                    if len(sel) else np.zeros(0, np.int64))
    else:
        new_rows = np.zeros(0, np.int64)
    # grown tracks keep refs in images outside this stage's bank: positions from
    # the feature store for those (few) keys
    ext_keys = np.fromiter((k for _, _, c in ext_jobs for k in c), np.int64)
    cam_ids = np.asarray(cams, np.int64)
    if len(new_rows):
        slot = np.searchsorted(bank.offsets, new_rows, side="right") - 1
        new_img = np.asarray(bank.image_ids, np.int64)[slot]
        new_pix = bank.host.xy.numpy()[new_rows].astype(np.float64).reshape(-1, 2)
    else:
        new_img, new_pix = np.zeros(0, np.int64), np.zeros((0, 2))
    ext_pix = np.array([feature_store.position(int(k) >> 32, int(k) & 0xFFFFFFFF)
                        for k in ext_keys], np.float64).reshape(-1, 2)
    cam = np.searchsorted(cam_ids, np.concatenate([new_img, ext_keys >> 32])).astype(np.int32)
    pix = np.concatenate([new_pix, ext_pix]).reshape(-1, 2)
    tracks = n_tr
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
