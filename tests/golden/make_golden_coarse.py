"""Golden fixtures for coarse unguided matching from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_coarse.py

* ``fransac_cases.npz``: estimate_fundamental_ransac (geometry.py:153-198) on
  synthetic two-view correspondences with outliers and noise (the style of
  test_geometry.py), per case the inlier mask, F, inlier count and planar flag.
* ``coarse_graph_*.npz``: build_coarse_matchgraph (matching.py:208-249) on the
  hold-out recipe (full tiers) and on a C1 scene with eta = 20 tiers; per edge
  the hybrid matches (query, target, f32 distance, ratio), F and inlier mask.
Scenes are stored by recipe and regenerated bit-identically on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))

from msfm.errors import InsufficientDataError  # noqa: E402
from msfm.geometry import estimate_fundamental_ransac  # noqa: E402
from msfm.matching import build_coarse_matchgraph, hybrid_match  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402


def fransac_cases():
    rng = np.random.default_rng(77)
    out = {}
    k = 0
    for n, outlier_frac, noise, planar in [(8, 0.0, 0.0, False), (12, 0.0, 0.2, False),
                                           (60, 0.3, 0.5, False), (300, 0.2, 0.3, False),
                                           (1000, 0.4, 0.5, False), (150, 0.6, 0.3, False),
                                           (2500, 0.1, 0.3, False), (200, 0.1, 0.2, True),
                                           (40, 0.5, 1.0, False), (7, 0.0, 0.0, False)]:
        K = np.array([[800.0, 0, 320], [0, 800.0, 240], [0, 0, 1]])
        X = rng.normal(size=(n, 3)) * np.array([1.5, 1.5, 0.0 if planar else 1.5])
        X += np.array([0, 0, 6.0])
        ang = rng.normal(size=3) * 0.15
        th = np.linalg.norm(ang)
        kx = ang / th
        Kx = np.array([[0, -kx[2], kx[1]], [kx[2], 0, -kx[0]], [-kx[1], kx[0], 0]])
        R = np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx
        t = np.array([1.0, 0.1, 0.05]) + rng.normal(size=3) * 0.05
        xq = X @ K.T
        uq = xq[:, :2] / xq[:, 2:3] + rng.normal(size=(n, 2)) * noise
        xc = (X @ R.T + t) @ K.T
        uc = xc[:, :2] / xc[:, 2:3] + rng.normal(size=(n, 2)) * noise
        m = int(round(outlier_frac * n))
        if m:
            uc[:m] = rng.uniform([0, 0], [640, 480], size=(m, 2))
        seed = int(rng.integers(0, 10000))
        out[f"c{k}_q"], out[f"c{k}_c"], out[f"c{k}_seed"] = uq, uc, np.array(seed)
        try:
            geom, mask = estimate_fundamental_ransac(uq, uc, seed=seed)
            out[f"c{k}_status"] = np.array("ok")
            out[f"c{k}_F"], out[f"c{k}_mask"] = geom.F, mask
            out[f"c{k}_count"] = np.array(geom.inlier_count)
            out[f"c{k}_planar"] = np.array(geom.degenerate_planar)
        except InsufficientDataError:
            out[f"c{k}_status"] = np.array("insufficient")
        except OverflowError:
            out[f"c{k}_status"] = np.array("overflow")   # geometry.py:189 quirk
        print("fransac case", k, n, str(out[f"c{k}_status"]),
              int(out[f"c{k}_count"]) if f"c{k}_count" in out else -1)
        k += 1
    out["n_cases"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "fransac_cases.npz"), **out)


def graph_fixture(name, spec_kw, eta=None):
    scene = generate_scene(SceneSpec(**spec_kw))
    store = scene.store()
    if eta is not None:
        store.apply_eta(eta)
    graph = build_coarse_matchgraph(store.sets)
    ids = sorted(store.sets)
    out = {"spec": np.array(repr(spec_kw)), "eta": np.array(-1.0 if eta is None else eta),
           "coarse": np.array([store.sets[i].coarse_count for i in ids])}
    keys = sorted(graph.edges)
    out["edges"] = np.array(keys, np.int32).reshape(-1, 2)
    for e, (a, b) in enumerate(keys):
        ed = graph.edges[(a, b)]
        out[f"e{e}_q"] = np.array([m.query.feature_id for m in ed.matches], np.int32)
        out[f"e{e}_t"] = np.array([m.target.feature_id for m in ed.matches], np.int32)
        out[f"e{e}_d"] = np.array([m.distance for m in ed.matches], np.float64)
        out[f"e{e}_r"] = np.array([m.ratio for m in ed.matches], np.float64)
        out[f"e{e}_F"] = ed.geometry.F
        out[f"e{e}_mask"] = ed.inlier_mask
        out[f"e{e}_count"] = np.array(ed.geometry.inlier_count)
    # hybrid_match of every pair (also the ones the graph drops), for the match lists
    hm = []
    for i, a in enumerate(ids):
        for b in ids[i + 1:]:
            ms = hybrid_match(store.sets[a], store.sets[b])
            hm.append((a, b, len(ms)))
    out["hybrid_counts"] = np.array(hm, np.int64).reshape(-1, 3)
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, "edges", len(keys), "pairs", len(hm))


if __name__ == "__main__":
    fransac_cases()
    graph_fixture("coarse_graph_holdout.npz", dict(n_cameras=12, n_points=700,
                                                   visibility_fraction=0.7, pixel_noise=0.3,
                                                   descriptor_noise=3.0, seed=77))
    graph_fixture("coarse_graph_c1eta.npz", dict(n_cameras=20, n_points=2000,
                                                 visibility_fraction=0.6, pixel_noise=0.5,
                                                 descriptor_noise=4.0, seed=1), eta=20.0)
