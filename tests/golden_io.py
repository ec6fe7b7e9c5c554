"""Load the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import ast
import hashlib
import os

import numpy as np

from paper_1512_06235_b200.synth import SceneSpec, generate_scene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_SCENES = {}


def scene_hash(scene) -> str:
    h = hashlib.sha256()
    for i in sorted(scene.feature_sets):
        fs = scene.feature_sets[i]
        h.update(fs.xy.tobytes()); h.update(fs.descriptors.tobytes())
    return h.hexdigest()[:16]


def load(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    kw = ast.literal_eval(str(z["spec"]))
    key = repr(sorted(kw.items()))
    if key not in _SCENES:
        _SCENES[key] = generate_scene(SceneSpec(**kw))
    scene = _SCENES[key]
    pairs = []
    for k in range(int(z["n_pairs"])):
        q, t = (int(v) for v in z[f"p{k}_qt"])
        qi = None if bool(z[f"p{k}_all"]) else z[f"p{k}_qi"].astype(np.int32)
        pairs.append(dict(q=q, t=t, qi=qi, mq=z[f"p{k}_mq"], mt=z[f"p{k}_mt"],
                          dist=z[f"p{k}_dist"], ratio=z[f"p{k}_ratio"], stats=z[f"p{k}_stats"]))
    return kw, scene, str(z["scene_hash"]), pairs


GUIDED_FIXTURES = sorted(f for f in os.listdir(GOLDEN) if f.startswith("guided_") and f.endswith(".npz"))
STRATEGY_FIXTURES = sorted(f for f in os.listdir(GOLDEN)
                           if f.startswith("strategy_") and f.endswith(".npz"))


def load_localize(name):
    """(spec kw, scene, snapshot, npz) of a localization fixture."""
    from paper_1512_06235_b200 import scenes

    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    kw = ast.literal_eval(str(z["spec"]))
    key = repr(sorted(kw.items()))
    if key not in _SCENES:
        _SCENES[key] = generate_scene(SceneSpec(**kw))
    scene = _SCENES[key]
    eta = float(z["eta"])
    snap = scenes.coarse_snapshot(scene, [int(i) for i in z["registered"]],
                                  eta=None if eta < 0 else eta)
    return kw, scene, snap, z
