"""The densify_stage drop-in reproduces the reference stage: same pairs, match
count, new points (ids and tracks), extended tracks; positions within 1e-6."""

import ast
import os

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["densify_C1.npz", "densify_ring12.npz"])
def test_densify_stage_equals_reference(name):
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.densify import densify_stage
    from paper_1512_06235_b200.synth import SceneSpec, generate_scene

    z = np.load(os.path.join(GOLDEN, name))
    scene = generate_scene(SceneSpec(**ast.literal_eval(str(z["spec"]))))
    snap = scenes.coarse_snapshot(scene, [int(i) for i in z["registered"]])
    model = scenes.snapshot_to_model(scene, snap)
    assert len(model.points) == int(z["n_before"])
    qi = [int(i) for i in z["query_images"]]
    summary = densify_stage(model, scene.store(), query_images=None if qi == [-1] else qi)
    assert [summary[k] for k in ("pairs", "matches", "new_points", "extended_tracks")] == \
        z["summary"].tolist()
    pids = sorted(model.points)
    assert pids == z["pids"].tolist()
    ptr, obs = z["ptr"], z["obs"]
    for j, p in enumerate(pids):
        assert sorted(model.points[p].track.items()) == [tuple(x) for x in obs[ptr[j]:ptr[j + 1]].tolist()]
    X = np.stack([model.points[p].position for p in pids])
    np.testing.assert_allclose(X, z["X"], rtol=1e-6, atol=1e-9)
