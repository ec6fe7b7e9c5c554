"""Golden fixtures for multi-view triangulation from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_tri.py

Tracks are the ones densify_stage triangulates on the C1 scene (guided
matches of every densify pair -> merge_tracks, densify.py:238-276), plus
hand-made edge cases in the style of test_geometry.py:293-379.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

from make_golden import coarse_model, densify_inputs  # noqa: E402
from msfm.densify import merge_tracks  # noqa: E402
from msfm.errors import DegenerateGeometryError  # noqa: E402
from msfm.geometry import fundamental_from_poses, triangulate_track  # noqa: E402
from msfm.guided import guided_match_pair  # noqa: E402
from msfm.model import Camera  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402


def tri(obs):
    try:
        r = triangulate_track(obs)
    except DegenerateGeometryError:
        return "degenerate", None, None
    if r is None:
        return "rejected", None, None
    return "ok", r.point, r.mean_error


def main():
    kw = dict(n_cameras=20, n_points=2000, visibility_fraction=0.6, pixel_noise=0.5,
              descriptor_noise=4.0, seed=1)
    scene = generate_scene(SceneSpec(**kw))
    model = coarse_model(scene, range(20))
    items = densify_inputs(model, scene)
    matches = []
    for q, t, qi in items:
        geom = fundamental_from_poses(scene.cameras[q], scene.cameras[t])
        matches.extend(guided_match_pair(scene.feature_sets[q], scene.feature_sets[t], geom,
                                         query_indices=qi))
    new_tracks, extensions = merge_tracks(matches, model)
    tracks = [[(r.image_id, r.feature_id) for r in refs] for refs in new_tracks]
    for pid in sorted(extensions):
        fresh = [r for r in sorted(set(extensions[pid]))
                 if model.owner(r) is None and r.image_id not in model.points[pid].track]
        if fresh:
            tracks.append([(r.image_id, r.feature_id) for r in model.points[pid].refs() + fresh])
    out = {"spec": np.array(repr(kw)), "n_tracks": np.array(len(tracks))}
    ptr = [0]
    flat = []
    status, X, err = [], [], []
    for tr in tracks:
        flat.extend(tr)
        ptr.append(len(flat))
        obs = [(scene.cameras[i], scene.feature_sets[i].xy[f].astype(np.float64)) for i, f in tr]
        s, x, e = tri(obs)
        status.append(s)
        X.append(x if x is not None else np.full(3, np.nan))
        err.append(e if e is not None else np.nan)
    out["ptr"] = np.array(ptr, np.int64)
    out["obs"] = np.array(flat, np.int32).reshape(-1, 2)
    out["status"] = np.array(status)
    out["X"] = np.array(X)
    out["err"] = np.array(err)
    out["n_matches"] = np.array(len(matches))
    # edge cases: explicit cameras/pixels
    rng = np.random.default_rng(7)
    K = np.array([[900.0, 0, 512], [0, 900.0, 384], [0, 0, 1]])

    def cam(C, look, iid):
        f = look - C
        f = f / np.linalg.norm(f)
        up = np.array([0.0, 0.0, 1.0])
        r = np.cross(f, up); r /= np.linalg.norm(r)
        R = np.stack([r, np.cross(f, r), f])
        return Camera(K=K, R=R, t=-R @ C, image_id=iid)

    cases = []
    Xw = np.array([0.2, -0.1, 0.3])
    for baseline, noise in [(2.0, 0.0), (2.0, 0.5), (0.05, 0.0), (0.01, 0.3), (3.0, 3.0)]:
        cams = [cam(np.array([-6.0, -baseline / 2, 0.2]), np.zeros(3), 0),
                cam(np.array([-6.0, baseline / 2, 0.2]), np.zeros(3), 1),
                cam(np.array([-5.5, 0.3, 1.0]), np.zeros(3), 2)]
        for nv in (2, 3):
            obs = []
            for c in cams[:nv]:
                p, _ = c.project(Xw)
                obs.append((c, p[0] + rng.normal(size=2) * noise))
            cases.append(obs)
    c0 = cam(np.array([-6.0, 0.0, 0.0]), np.zeros(3), 0)
    cases.append([(c0, np.array([500.0, 400.0])), (c0, np.array([520.0, 380.0]))])   # same centre
    cb = cam(np.array([6.0, 0.0, 0.0]), np.zeros(3), 1)
    pa, _ = c0.project(Xw)
    cases.append([(c0, pa[0]), (cb, np.array([-4000.0, 9000.0]))])                     # wild pixel
    for k, obs in enumerate(cases):
        s, x, e = tri(obs)
        out[f"e{k}_K"] = np.stack([o[0].K for o in obs])
        out[f"e{k}_R"] = np.stack([o[0].R for o in obs])
        out[f"e{k}_t"] = np.stack([o[0].t for o in obs])
        out[f"e{k}_pix"] = np.stack([o[1] for o in obs])
        out[f"e{k}_status"] = np.array(s)
        if x is not None:
            out[f"e{k}_X"], out[f"e{k}_err"] = x, np.array(e)
    out["n_edges"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "triangulate.npz"), **out)
    print("tracks", len(tracks), "matches", len(matches), "status",
          {s: status.count(s) for s in set(status)}, "edge", [str(out[f'e{k}_status']) for k in range(len(cases))])


if __name__ == "__main__":
    main()
