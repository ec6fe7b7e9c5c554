"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container only (needs /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference is imported read-only from MSFM_REF_PATH (default
/root/reference/pkg/src).  Fixtures store the scene recipe (regenerated
bit-identically by paper_1512_06235_b200.synth, pinned by a content hash) and
the reference's outputs, so they stay small and travel to the GPU box.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))
sys.path.insert(0, REPO)

from msfm import densify as rdensify  # noqa: E402
from msfm.descriptors import SearchStats  # noqa: E402
from msfm.geometry import fundamental_from_poses  # noqa: E402
from msfm.guided import guided_match_pair  # noqa: E402
from msfm.model import FeatureRef, Model  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402


def scene_hash(scene) -> str:
    h = hashlib.sha256()
    for i in sorted(scene.feature_sets):
        fs = scene.feature_sets[i]
        h.update(fs.xy.tobytes()); h.update(fs.descriptors.tobytes())
    return h.hexdigest()[:16]


def coarse_model(scene, registered, eta=20.0):
    """SURVEY.md Appendix B M0 recipe with the reference's own classes."""
    store = scene.store()
    store.apply_eta(eta)
    gt = scene.ground_truth_model()
    model = Model(stage_tag="coarse")
    for i in sorted(registered):
        model.attach_camera(gt.cameras[i])
    for pid in gt.point_ids():
        refs = [FeatureRef(i, f) for i, f in sorted(gt.points[pid].track.items())
                if i in model.cameras and f < store.sets[i].coarse_count]
        if len(refs) >= 2:
            model.add_point(gt.points[pid].position, refs)
    return model


def densify_inputs(model, scene):
    """The pair list / roles / untracked sets densify_stage builds (densify.py:186-207)."""
    registered = model.image_ids()
    k_limit = max(1, int(np.ceil(0.10 * len(registered))))
    sets = []
    for i in registered:
        cs = rdensify.candidate_images(model, i, threshold=8, k_limit=k_limit)
        if cs.candidates:
            sets.append(cs)
    pairs = rdensify.unique_pairs(sets)
    out = []
    for a, b in pairs:
        q, t = a, b  # every registered image is a query image
        fs = scene.feature_sets[q]
        owned = [f for f in range(len(fs)) if model.owner(FeatureRef(q, f)) is not None]
        mask = np.ones(len(fs), bool); mask[owned] = False
        out.append((q, t, np.flatnonzero(mask)))
    return out


def run_pairs(scene, items, **kw):
    rows = []
    for q, t, qi in items:
        geom = fundamental_from_poses(scene.cameras[q], scene.cameras[t])
        st = SearchStats()
        ms = guided_match_pair(scene.feature_sets[q], scene.feature_sets[t], geom,
                               query_indices=qi, stats=st, **kw)
        rows.append(dict(q=q, t=t, qi=np.asarray(qi, np.int32) if qi is not None else None,
                         mq=np.array([m.query.feature_id for m in ms], np.int32),
                         mt=np.array([m.target.feature_id for m in ms], np.int32),
                         dist=np.array([m.distance for m in ms], np.float64),
                         ratio=np.array([m.ratio for m in ms], np.float64),
                         stats=np.array([st.queries, st.candidates], np.int64)))
    return rows


def save(name, spec_kw, scene, rows, extra=None):
    payload = {"spec": np.array(repr(spec_kw)), "scene_hash": np.array(scene_hash(scene)),
               "n_pairs": np.array(len(rows))}
    for k, r in enumerate(rows):
        payload[f"p{k}_qt"] = np.array([r["q"], r["t"]], np.int32)
        payload[f"p{k}_qi"] = r["qi"] if r["qi"] is not None else np.array([-1], np.int32)
        payload[f"p{k}_all"] = np.array(r["qi"] is None)
        for key in ("mq", "mt", "dist", "ratio", "stats"):
            payload[f"p{k}_{key}"] = r[key]
    if extra:
        payload.update(extra)
    np.savez_compressed(os.path.join(HERE, name), **payload)
    print(name, len(rows), "pairs,", sum(len(r["mq"]) for r in rows), "matches")


def main():
    # 1. reference unit-test scenes (test_guided.py:256-335): full query sets
    for seed in range(9, 15):
        kw = dict(n_cameras=2, layout="grid", ring_radius=1.2, cloud_radius=2.0,
                  n_points=600, seed=seed)
        sc = generate_scene(SceneSpec(**kw))
        save(f"guided_unit_s{seed}.npz", kw, sc, run_pairs(sc, [(0, 1, None), (1, 0, None)]))
    kw = dict(n_cameras=2, layout="grid", ring_radius=1.2, cloud_radius=2.0, n_points=500,
              seed=12, repetition_groups=20, repetition_group_size=10, descriptor_noise=2.0,
              pixel_noise=0.3)
    sc = generate_scene(SceneSpec(**kw))
    save("guided_repetition.npz", kw, sc, run_pairs(sc, [(0, 1, None), (1, 0, None)]))
    # edge cases: single query (dgemv line path), empty query list, tiny subsets
    sc = generate_scene(SceneSpec(n_cameras=3, n_points=400, seed=5))
    items = [(0, 1, np.array([7])), (0, 1, np.array([], np.int64)), (1, 2, np.arange(0, 60, 3)),
             (2, 0, np.array([0, 1])), (1, 0, None)]
    save("guided_edges.npz", dict(n_cameras=3, n_points=400, seed=5), sc, run_pairs(sc, items))

    # 2. C1 (configs[0]): every densify pair of the 20-camera scene
    kw = dict(n_cameras=20, n_points=2000, visibility_fraction=0.6, pixel_noise=0.5,
              descriptor_noise=4.0, seed=1)
    sc = generate_scene(SceneSpec(**kw))
    model = coarse_model(sc, range(20))
    items = densify_inputs(model, sc)
    save("guided_C1.npz", kw, sc, run_pairs(sc, items))

    # 3. 8k-feature pairs (C2/C3 scene recipe, 10 cameras): the benchmark's feature density
    kw = dict(n_cameras=10, n_points=12000, image_width=3072, image_height=2304, focal=2600.0,
              visibility_fraction=0.55, clutter_per_image=2700, pixel_noise=0.5,
              descriptor_noise=4.0, seed=2)
    sc = generate_scene(SceneSpec(**kw))
    model = coarse_model(sc, range(10))
    items = densify_inputs(model, sc)[:6]
    save("guided_8k.npz", kw, sc, run_pairs(sc, items))


def strategies():
    """guided_match_pair with strategy="linear" / "radial" (guided.py:190-194,
    273-285, 425-431) on the unit scenes, the edge cases, C1 pairs and two 8k pairs."""
    for strat in ("linear", "radial"):
        rows_all = []
        scenes_kw = []
        for seed in (9, 10):
            kw = dict(n_cameras=2, layout="grid", ring_radius=1.2, cloud_radius=2.0,
                      n_points=600, seed=seed)
            sc = generate_scene(SceneSpec(**kw))
            save(f"strategy_{strat}_s{seed}.npz", kw, sc,
                 run_pairs(sc, [(0, 1, None), (1, 0, None)], strategy=strat))
        sc = generate_scene(SceneSpec(n_cameras=3, n_points=400, seed=5))
        items = [(0, 1, np.array([7])), (0, 1, np.array([], np.int64)),
                 (1, 2, np.arange(0, 60, 3)), (2, 0, np.array([0, 1])), (1, 0, None)]
        save(f"strategy_{strat}_edges.npz", dict(n_cameras=3, n_points=400, seed=5), sc,
             run_pairs(sc, items, strategy=strat))
        kw = dict(n_cameras=20, n_points=2000, visibility_fraction=0.6, pixel_noise=0.5,
                  descriptor_noise=4.0, seed=1)
        sc = generate_scene(SceneSpec(**kw))
        model = coarse_model(sc, range(20))
        items = densify_inputs(model, sc)[::4]
        save(f"strategy_{strat}_C1.npz", kw, sc, run_pairs(sc, items, strategy=strat))
        kw = dict(n_cameras=10, n_points=12000, image_width=3072, image_height=2304, focal=2600.0,
                  visibility_fraction=0.55, clutter_per_image=2700, pixel_noise=0.5,
                  descriptor_noise=4.0, seed=2)
        sc = generate_scene(SceneSpec(**kw))
        model = coarse_model(sc, range(10))
        items = densify_inputs(model, sc)[:2]
        save(f"strategy_{strat}_8k.npz", kw, sc, run_pairs(sc, items, strategy=strat))


if __name__ == "__main__":
    if sys.argv[1:] == ["strategies"]:
        strategies()
    else:
        main()
