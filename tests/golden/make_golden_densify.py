"""Golden fixture for the whole point-addition stage from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_densify.py

Runs msfm.densify.densify_stage (densify.py:168-286) on the C1 scene's coarse
model M0 and on a 12-camera scene; stores the summary and every resulting
point (id, track, position).
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

from make_golden import coarse_model  # noqa: E402
from msfm.densify import densify_stage  # noqa: E402
from msfm.synth import SceneSpec, generate_scene  # noqa: E402


def run(name, kw, registered, query_images=None):
    scene = generate_scene(SceneSpec(**kw))
    model = coarse_model(scene, registered)
    n0 = len(model.points)
    summary = densify_stage(model, scene.store(), query_images=query_images)
    pids = sorted(model.points)
    ptr = [0]
    obs = []
    for p in pids:
        obs.extend(sorted(model.points[p].track.items()))
        ptr.append(len(obs))
    np.savez_compressed(os.path.join(HERE, name), spec=np.array(repr(kw)),
                        registered=np.array(sorted(registered)),
                        query_images=np.array(query_images if query_images is not None else [-1]),
                        summary=np.array([summary[k] for k in ("pairs", "matches", "new_points",
                                                              "extended_tracks")]),
                        n_before=np.array(n0), pids=np.array(pids), ptr=np.array(ptr),
                        obs=np.array(obs, np.int32).reshape(-1, 2),
                        X=np.stack([model.points[p].position for p in pids]))
    print(name, summary, "points", n0, "->", len(pids))


if __name__ == "__main__":
    run("densify_C1.npz", dict(n_cameras=20, n_points=2000, visibility_fraction=0.6,
                               pixel_noise=0.5, descriptor_noise=4.0, seed=1), range(20))
    # 1500 features/img so the eta=20 tier leaves most features untracked
    run("densify_ring12.npz", dict(n_cameras=12, n_points=2500, visibility_fraction=0.55,
                                   pixel_noise=0.4, descriptor_noise=3.0, clutter_per_image=300,
                                   seed=31), range(12), query_images=[0, 3, 4, 9])
