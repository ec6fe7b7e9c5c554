"""Golden fixtures for 3D-2D localization and PnP-RANSAC from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_localize.py

For each held-out image the reference's own functions run with the exact kNN
index (DescriptorIndex(exact_threshold=10**9), the parity path of SURVEY.md
§8c): knn2 of the point mean descriptors (descriptors.py:35-72),
direct_3d2d_search (localize.py:99-122) and pnp_ransac(seed=image_id)
(reconstruct.py:168-226).  The model is described by its recipe so the scene
is regenerated bit-identically on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))
sys.path.insert(0, REPO)

from msfm.descriptors import DescriptorIndex  # noqa: E402
from msfm.localize import direct_3d2d_search, mean_descriptor  # noqa: E402
from msfm.model import FeatureRef, Model  # noqa: E402
from msfm.reconstruct import pnp_ransac  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402


def partial_model(scene, registered, eta=None):
    """GT points restricted to registered cameras (and coarse tier if eta)."""
    store = scene.store()
    if eta is not None:
        store.apply_eta(eta)
    gt = scene.ground_truth_model()
    model = Model(stage_tag="coarse")
    for i in sorted(registered):
        model.attach_camera(gt.cameras[i])
    for pid in gt.point_ids():
        refs = [FeatureRef(i, f) for i, f in sorted(gt.points[pid].track.items())
                if i in model.cameras and (eta is None or f < store.sets[i].coarse_count)]
        if len(refs) >= 2:
            model.add_point(gt.points[pid].position, refs)
    return model


def run(name, spec_kw, registered, queries, eta=None):
    scene = generate_scene(SceneSpec(**spec_kw))
    store = scene.store()
    model = partial_model(scene, registered, eta)
    pids = sorted(model.points)
    Q = np.stack([mean_descriptor(model.points[p], store) for p in pids])
    out = {"spec": np.array(repr(spec_kw)), "registered": np.array(sorted(registered)),
           "eta": np.array(-1.0 if eta is None else eta), "queries": np.array(queries),
           "n_points": np.array(len(pids))}
    for q in queries:
        fs = store.sets[q]
        index = DescriptorIndex(fs.descriptors_f32(), exact_threshold=10**9)
        dist, idx = index.knn2(Q)
        corr = direct_3d2d_search(model, pids, fs, store, index=index)
        out[f"q{q}_knn_idx"] = idx.astype(np.int32)
        out[f"q{q}_knn_dist"] = dist
        c = np.array(corr, dtype=np.int32).reshape(-1, 2)
        out[f"q{q}_corr"] = c
        res, status = None, "below_gate"
        if len(c) > 16:
            X = np.stack([model.points[p].position for p, _ in corr])
            uv = np.stack([fs.xy[f] for _, f in corr]).astype(np.float64)
            try:
                res = pnp_ransac(X, uv, scene.cameras[q].K, seed=q)
                status = "ok" if res is not None else "none"
            except OverflowError:
                status = "overflow"   # reconstruct.py:210-211 quirk
        out[f"q{q}_ok"] = np.array(res is not None)
        out[f"q{q}_status"] = np.array(status)
        if res is not None:
            R, t, mask = res
            out[f"q{q}_R"], out[f"q{q}_t"], out[f"q{q}_mask"] = R, t, mask
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, "points", len(pids), "queries", len(queries),
          "corr", [int(len(out[f"q{q}_corr"])) for q in queries],
          "status", [str(out[f"q{q}_status"]) for q in queries])


def pnp_cases():
    """Direct pnp_ransac cases in the style of test_reconstruct.py:23-83."""
    rng = np.random.default_rng(2024)
    out = {}
    k = 0
    for n, outlier_frac, noise in [(6, 0.0, 0.0), (40, 0.0, 0.0), (200, 0.4, 0.5), (800, 0.2, 0.3),
                                   (3000, 0.05, 0.3), (60, 0.3, 1.0), (500, 0.6, 0.3),
                                   (1500, 0.1, 0.2)]:
        K = np.array([[900.0, 0, 512], [0, 900.0, 384], [0, 0, 1]])
        ang = rng.normal(size=3) * 0.3
        th = np.linalg.norm(ang)
        kx = ang / th
        Kx = np.array([[0, -kx[2], kx[1]], [kx[2], 0, -kx[0]], [-kx[1], kx[0], 0]])
        R = np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx
        t = rng.normal(size=3) * 0.5 + np.array([0, 0, 6.0])
        X = rng.normal(size=(n, 3)) * 1.5
        xc = X @ R.T + t
        uv = (xc @ K.T)[:, :2] / xc[:, 2:3] + rng.normal(size=(n, 2)) * noise
        m = int(round(outlier_frac * n))
        if m:
            uv[:m] = rng.uniform([0, 0], [1024, 768], size=(m, 2))
        seed = int(rng.integers(0, 1000))
        try:
            res = pnp_ransac(X, uv, K, seed=seed)
            status = "ok" if res is not None else "none"
        except OverflowError:
            res, status = None, "overflow"
        out[f"c{k}_X"], out[f"c{k}_uv"], out[f"c{k}_K"] = X, uv, K
        out[f"c{k}_seed"] = np.array(seed)
        out[f"c{k}_status"] = np.array(status)
        if res is not None:
            out[f"c{k}_R"], out[f"c{k}_t"], out[f"c{k}_mask"] = res
        print("pnp case", k, n, outlier_frac, status)
        k += 1
    out["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "pnp_cases.npz"), **out)


def ranked_cases():
    """ranked_2d2d_search (localize.py:125-176) on the hold-out recipe of
    test_localize.py:18-38, exact index, plus the copied-image case of
    test_localize.py:201-221 and the below-gate case."""
    import dataclasses

    from msfm.matching import Edge, Match, MatchGraph, build_coarse_matchgraph
    from msfm.localize import ranked_2d2d_search

    kw = dict(n_cameras=12, n_points=700, visibility_fraction=0.7, pixel_noise=0.3,
              descriptor_noise=3.0, seed=77)
    scene = generate_scene(SceneSpec(**kw))
    store = scene.store()
    graph = build_coarse_matchgraph(store.sets)
    model = partial_model(scene, range(9))
    out = {"spec": np.array(repr(kw)), "registered": np.arange(9), "eta": np.array(-1.0)}
    edges = sorted(graph.edges)
    out["edges"] = np.array([[a, b, len(graph.edges[(a, b)].matches)] for a, b in edges], np.int64)
    for q in (9, 10, 11):
        fs = store.sets[q]
        idx = DescriptorIndex(fs.descriptors_f32(), exact_threshold=10**9)
        corr = ranked_2d2d_search(model, graph, q, fs, store, index=idx)
        out[f"r{q}_corr"] = np.array(corr, dtype=np.int32).reshape(-1, 2)
        strict = ranked_2d2d_search(model, graph, q, fs, store, ratio=1e-6,
                                    index=DescriptorIndex(fs.descriptors_f32(), exact_threshold=10**9))
        out[f"r{q}_strict_n"] = np.array(len(strict))
    source = model.image_ids()[0]
    fs = dataclasses.replace(store[source], image_id=97)
    g = MatchGraph()
    key = (min(97, source), max(97, source))
    g.edges[key] = Edge(matches=[Match(query=FeatureRef(key[0], i), target=FeatureRef(key[1], i),
                                       distance=0.0, ratio=0.0) for i in range(40)])
    corr = ranked_2d2d_search(model, g, 97, fs, store,
                              index=DescriptorIndex(fs.descriptors_f32(), exact_threshold=10**9))
    out["copy_source"] = np.array(source)
    out["copy_corr"] = np.array(corr, dtype=np.int32).reshape(-1, 2)
    np.savez_compressed(os.path.join(HERE, "localize_ranked.npz"), **out)
    print("ranked", {q: len(out[f"r{q}_corr"]) for q in (9, 10, 11)}, "copy", len(corr))


def setcover_cases():
    """compute_set_cover (localize.py:62-96) on seeded models, several k, and the
    forced set-cover path of localize_all (test_localize.py:289-295) on the
    hold-out recipe."""
    import copy

    from msfm.localize import compute_set_cover, localize_all
    from msfm.matching import MatchGraph

    out = {}
    cases = [dict(n_cameras=4, n_points=30, seed=13), dict(n_cameras=8, n_points=200, seed=7),
             dict(n_cameras=12, n_points=700, visibility_fraction=0.7, seed=77),
             dict(n_cameras=30, n_points=2500, visibility_fraction=0.6, seed=5)]
    ks = [1, 3, 5, 40, 10_000]
    for c, kw in enumerate(cases):
        scene = generate_scene(SceneSpec(**kw))
        model = partial_model(scene, range(kw["n_cameras"]))
        out[f"c{c}_spec"] = np.array(repr(kw))
        for k in ks:
            cov = compute_set_cover(model, k)
            out[f"c{c}_k{k}_selected"] = np.array(cov.selected, np.int64)
            out[f"c{c}_k{k}_coverage"] = np.array(list(cov.coverage.items()), np.int64).reshape(-1, 2)
    out["n_cases"] = np.array(len(cases))
    out["ks"] = np.array(ks)
    kw = dict(n_cameras=12, n_points=700, visibility_fraction=0.7, pixel_noise=0.3,
              descriptor_noise=3.0, seed=77)
    scene = generate_scene(SceneSpec(**kw))
    store = scene.store()
    model = copy.deepcopy(partial_model(scene, range(9)))
    K = {i: scene.cameras[i].K for i in store.sets}
    cover = compute_set_cover(model, 40).selected
    newly, results = localize_all(model, store, MatchGraph(), K, force_set_cover=True,
                                  set_cover_k=40)
    out["forced_spec"] = np.array(repr(kw))
    out["forced_cover"] = np.array(cover, np.int64)
    out["forced_newly"] = np.array(newly, np.int64)
    for r in results:
        q = r.image_id
        out[f"forced_q{q}_corr"] = np.array(r.correspondences, np.int32).reshape(-1, 2)
        out[f"forced_q{q}_method"] = np.array(r.method)
        if r.pose is not None:
            out[f"forced_q{q}_R"], out[f"forced_q{q}_t"] = r.pose.R, r.pose.t
            out[f"forced_q{q}_inliers"] = np.array(r.inliers)
    np.savez_compressed(os.path.join(HERE, "setcover.npz"), **out)
    print("setcover", {k: len(out[f"c3_k{k}_selected"]) for k in ks}, "forced newly", newly,
          "cover", len(cover))


if __name__ == "__main__":
    if sys.argv[1:] == ["setcover"]:
        setcover_cases()
        sys.exit(0)
    if sys.argv[1:] == ["ranked"]:
        ranked_cases()
        sys.exit(0)
    # reference unit-test style hold-out (test_localize.py:18-38): last 3 cameras removed
    run("localize_holdout.npz", dict(n_cameras=12, n_points=700, visibility_fraction=0.7,
                                     pixel_noise=0.3, descriptor_noise=3.0, seed=77),
        registered=range(9), queries=[9, 10, 11])
    # C2 recipe at 8k features/img, 30 cameras, every 5th registered, tier-only M0
    run("localize_c2mini.npz", dict(n_cameras=30, n_points=12000, image_width=3072,
                                    image_height=2304, focal=2600.0, visibility_fraction=0.55,
                                    clutter_per_image=2700, pixel_noise=0.5, descriptor_noise=4.0,
                                    seed=2),
        registered=range(0, 30, 5), queries=[1, 2, 3, 4, 7, 8, 13, 21, 29], eta=20.0)
    pnp_cases()
