"""GPU parity of the tcgen05 kNN and the direct 3D-2D search (through the C-ABI)."""

import numpy as np
import pytest

from golden_io import load_localize
from oracle import localize as ol

pytestmark = pytest.mark.gpu


def _random_case(rng, M, sizes, max_n=10, dup=False, any_sum=False, min_n=1):
    from paper_1512_06235_b200.types import FeatureSet
    sets = {}
    for i, nf in enumerate(sizes):
        desc = rng.integers(0, 256, size=(nf, 128), dtype=np.uint8)
        if dup and nf > 4:
            desc[3] = desc[1]          # exact ties: lowest index must win
        sets[i] = FeatureSet(image_id=i, width=640, height=480,
                             xy=rng.uniform(0, 400, size=(nf, 2)).astype(np.float32),
                             scale=np.ones(nf, np.float32), orientation=np.zeros(nf, np.float32),
                             descriptors=desc)
    n = rng.integers(min_n, max_n + 1, size=M).astype(np.int32)
    if any_sum:
        # any track sum a track of n uint8 rows can have (every digit of 2S exercised)
        S = (rng.random((M, 128)) * (255 * n[:, None] + 1)).astype(np.int64).astype(np.int32)
    else:
        S = (rng.integers(0, 256, size=(M, 128)) * n[:, None]).astype(np.int32)
    if dup and M > 3:
        S[2] = S[0] if n[2] == n[0] else S[2]
    return sets, S, n


@pytest.mark.parametrize("M,sizes,max_n,any_sum,min_n",
                         [(1, [1], 1, False, 1), (5, [3, 1, 0, 130], 4, False, 1),
                          (128, [128], 10, False, 1), (300, [257, 1000, 5], 10, False, 1),
                          (1000, [2000, 129], 100, False, 1), (200, [16000, 31], 12, False, 1),
                          # long tracks (C5's coarse model): three digit planes, int64 keys,
                          # mixed with short ones in the same call
                          (700, [3000, 64], 3000, True, 1), (300, [1500], 32767, True, 101),
                          (257, [16000], 600, True, 90)])
def test_knn_topk_matches_exact_oracle(M, sizes, max_n, any_sum, min_n):
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.localize import PointSet, knn2_tracks

    rng = np.random.default_rng(M + len(sizes))
    sets, S, n = _random_case(rng, M, sizes, max_n, dup=True, any_sum=any_sum, min_n=min_n)
    bank = FeatureBank(sets)
    pts = PointSet(S=S, n=n, ids=np.arange(M))
    imgs = [i for i in sets]
    res = knn2_tracks(bank, pts, imgs)
    for s, i in enumerate(imgs):
        F = sets[i].descriptors
        idx, nb, ns = res.host(pts, s)
        if len(F) == 0:
            assert (idx == -1).all()
            continue
        oi, onb, ons = ol.knn2_exact(S, n, F)
        np.testing.assert_array_equal(idx, oi)
        np.testing.assert_array_equal(nb, onb)
        np.testing.assert_array_equal(ns, ons)
    if max_n > 100:
        # the direct 3D-2D search on long tracks (int64 keys end to end)
        from paper_1512_06235_b200.localize import direct_search
        big = [i for i in imgs if len(sets[i].descriptors) > 1]
        corr = direct_search(bank, pts, big)
        for c, i in zip(corr, big):
            np.testing.assert_array_equal(c, ol.direct_3d2d(np.arange(M), S, n, sets[i].descriptors))


@pytest.mark.parametrize("name", ["localize_holdout.npz", "localize_c2mini.npz"])
def test_direct_search_equals_reference(name):
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.localize import PointSet, direct_search
    from paper_1512_06235_b200 import scenes

    kw, scene, snap, z = load_localize(name)
    S, n = scenes.track_sums(scene, snap)
    pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
    bank = FeatureBank(scene.feature_sets)
    qs = [int(q) for q in z["queries"]]
    got = direct_search(bank, pts, qs)
    for s, q in enumerate(qs):
        np.testing.assert_array_equal(got[s], z[f"q{q}_corr"])


@pytest.mark.parametrize("name", ["localize_holdout.npz", "localize_c2mini.npz"])
def test_gather_pnp_inputs_equals_host_gather(name):
    """msfm_gather_3d2d: X / uv of the gated images == the host gather of the
    reference's correspondences (localize.py:203-211)."""
    import torch

    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.localize import PointSet, direct_search, gather_pnp_inputs
    from paper_1512_06235_b200 import scenes

    kw, scene, snap, z = load_localize(name)
    S, n = scenes.track_sums(scene, snap)
    pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
    qs = [int(q) for q in z["queries"]]
    bank = FeatureBank({q: scene.feature_sets[q] for q in qs})
    corr = direct_search(bank, pts, qs, to_host=False)
    d_xyz = torch.from_numpy(np.ascontiguousarray(snap.point_xyz)).cuda()
    for gate in (16, 0, 10**9):
        X, uv, off, todo = gather_pnp_inputs(bank, corr, qs, d_xyz, gate=gate)
        want = [k for k, q in enumerate(qs) if len(z[f"q{q}_corr"]) > gate]
        assert todo.tolist() == want
        X, uv = X.cpu().numpy(), uv.cpu().numpy()
        for j, k in enumerate(todo):
            c = z[f"q{qs[k]}_corr"]
            np.testing.assert_array_equal(X[off[j]:off[j + 1]], snap.point_xyz[c[:, 0]])
            np.testing.assert_array_equal(uv[off[j]:off[j + 1]],
                                          scene.feature_sets[qs[k]].xy[c[:, 1]].astype(np.float64))


class _NoGraph:
    def neighbors(self, image_id):
        return []

    def match_count(self, a, b):
        return 0


def test_localize_all_equals_reference_holdout():
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.localize import localize_all

    kw, scene, snap, z = load_localize("localize_holdout.npz")
    model = scenes.snapshot_to_model(scene, snap)
    store = scene.store()
    K = {i: scene.cameras[i].K for i in store.sets}
    newly, results = localize_all(model, store, _NoGraph(), K)
    qs = [int(q) for q in z["queries"]]
    assert newly == [q for q in qs if str(z[f"q{q}_status"]) == "ok"]
    for r in results:
        q = r.image_id
        assert [tuple(c) for c in z[f"q{q}_corr"].tolist()] == r.correspondences
        np.testing.assert_allclose(r.pose.R, z[f"q{q}_R"], atol=1e-6)
        np.testing.assert_allclose(r.pose.t, z[f"q{q}_t"], atol=1e-6, rtol=1e-6)
        assert r.inliers == int(z[f"q{q}_mask"].sum())
        assert model.is_registered(q)
    assert model.stage_tag == "after_localize(1)"


def test_localize_all_raises_like_reference_on_overflow():
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.localize import localize_all

    kw, scene, snap, z = load_localize("localize_c2mini.npz")
    model = scenes.snapshot_to_model(scene, snap)
    store = scene.store()
    store.sets = {q: store.sets[q] for q in list(z["registered"]) + [int(x) for x in z["queries"]]}
    K = {i: scene.cameras[i].K for i in store.sets}
    with pytest.raises(OverflowError):
        localize_all(model, store, _NoGraph(), K)


class _EdgeGraph:
    """MatchGraph stand-in carrying the reference graph's edge counts."""

    def __init__(self, edges):
        self.count = {(int(a), int(b)): int(c) for a, b, c in edges}

    def neighbors(self, image_id):
        return sorted([b for a, b in self.count if a == image_id] +
                      [a for a, b in self.count if b == image_id])

    def match_count(self, a, b):
        return self.count.get((min(a, b), max(a, b)), 0)


def test_ranked_2d2d_equals_reference():
    """ranked_2d2d_search (localize.py:125-176) through the device kNN: same
    correspondences as the reference with its exact index."""
    import dataclasses

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.localize import ranked_2d2d_search
    from paper_1512_06235_b200.types import InsufficientDataError

    kw, scene, snap, z = load_localize("localize_ranked.npz")
    model = scenes.snapshot_to_model(scene, snap)
    store = scene.store()
    graph = _EdgeGraph(z["edges"])
    for q in (9, 10, 11):
        corr = ranked_2d2d_search(model, graph, q, store.sets[q], store)
        assert [tuple(c) for c in z[f"r{q}_corr"].tolist()] == corr
        strict = ranked_2d2d_search(model, graph, q, store.sets[q], store, ratio=1e-6)
        assert len(strict) == int(z[f"r{q}_strict_n"]) == 0
    src = int(z["copy_source"])
    fs = dataclasses.replace(store.sets[src], image_id=97)
    g = _EdgeGraph([(min(97, src), max(97, src), 40)])
    corr = ranked_2d2d_search(model, g, 97, fs, store)
    assert [tuple(c) for c in z["copy_corr"].tolist()] == corr
    with pytest.raises(InsufficientDataError):
        ranked_2d2d_search(model, _EdgeGraph([]), 9, store.sets[9], store)


def test_staged_knn_equals_resident_knn():
    """knn2_tracks_staged (query bank uploaded in ranges, kNN per range as it lands)
    == knn2_tracks over a resident bank."""
    import torch

    from paper_1512_06235_b200.bank import FeatureBank, HostBank
    from paper_1512_06235_b200.localize import PointSet, knn2_tracks, knn2_tracks_staged, upload_points

    rng = np.random.default_rng(11)
    sets = {}
    for i in range(7):
        sets[i] = _random_case(rng, 1, [int(rng.integers(50, 900))])[0][0]
    S = rng.integers(0, 256, size=(300, 128)).astype(np.int32) * 2
    pts = PointSet(S=S, n=np.full(300, 2, np.int32), ids=np.arange(300))
    full = FeatureBank(sets)
    want = knn2_tracks(full, pts, list(range(7)))
    for groups in (1, 3, 7):
        b = FeatureBank(host=HostBank(sets), staged=True)
        got = knn2_tracks_staged(b, pts, list(range(7)), upload_points(pts, b.device), groups)
        torch.cuda.synchronize()
        for name in ("k1", "i1", "k2"):
            assert torch.equal(getattr(got, name)[:, :300], getattr(want, name)[:, :300]), (groups, name)


def test_localize_all_forced_set_cover_equals_reference():
    """localize_all(force_set_cover=True, set_cover_k=40) (test_localize.py:289-295):
    the cover, correspondences, poses and newly registered images equal the
    reference run recorded in setcover.npz."""
    import os

    from golden_io import GOLDEN
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.localize import compute_set_cover, localize_all
    from paper_1512_06235_b200.synth import SceneSpec, generate_scene

    z = np.load(os.path.join(GOLDEN, "setcover.npz"))
    scene = generate_scene(SceneSpec(**eval(str(z["forced_spec"]))))
    snap = scenes.coarse_snapshot(scene, range(9), eta=None)
    model = scenes.snapshot_to_model(scene, snap)
    store = scene.store()
    K = {i: scene.cameras[i].K for i in store.sets}
    assert compute_set_cover(model, 40).selected == z["forced_cover"].tolist()
    newly, results = localize_all(model, store, _NoGraph(), K, force_set_cover=True,
                                  set_cover_k=40)
    assert newly == z["forced_newly"].tolist()
    for r in results:
        q = r.image_id
        assert [tuple(c) for c in z[f"forced_q{q}_corr"].tolist()] == r.correspondences
        assert r.method == str(z[f"forced_q{q}_method"])
        if f"forced_q{q}_R" in z:
            np.testing.assert_allclose(r.pose.R, z[f"forced_q{q}_R"], atol=1e-6)
            np.testing.assert_allclose(r.pose.t, z[f"forced_q{q}_t"], atol=1e-6, rtol=1e-6)
            assert r.inliers == int(z[f"forced_q{q}_inliers"])


def test_track_sums_device_equals_host():
    """K7 (mean_descriptor localize.py:51-59 in exact integers): device sums over a
    track CSR equal numpy's, incl. long tracks, a single-view and an empty track;
    model_points (the drop-ins' path) equals the harness's host sums."""
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.localize import model_points, track_sums_device

    rng = np.random.default_rng(5)
    sets, _, _ = _random_case(rng, 1, [3000, 17, 900])
    bank = FeatureBank(sets)
    lens = np.array([0, 1, 7, 150, 2999, 3], np.int64)
    ptr = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    rows = rng.integers(0, bank.n_total, size=int(ptr[-1]))
    dS, dn, dSS = track_sums_device(bank, ptr, rows)
    D = np.concatenate([sets[i].descriptors for i in sorted(sets)]).astype(np.int64)
    want = np.stack([D[rows[ptr[p]:ptr[p + 1]]].sum(0) for p in range(len(lens))])
    np.testing.assert_array_equal(dS[:len(lens)].cpu().numpy(), want)
    np.testing.assert_array_equal(dn[:len(lens)].cpu().numpy(), lens)
    np.testing.assert_array_equal(dSS[:len(lens)].cpu().numpy(), (want * want).sum(1))
    kw, scene, snap, z = load_localize("localize_c2mini.npz")
    model = scenes.snapshot_to_model(scene, snap)
    pts = model_points(model, scene.store(), sorted(model.points))
    S, n = scenes.track_sums(scene, snap)
    np.testing.assert_array_equal(pts.dev[0][:len(n)].cpu().numpy(), S)
    np.testing.assert_array_equal(pts.n, n)
    np.testing.assert_array_equal(pts.SS, (S.astype(np.int64) ** 2).sum(1))
