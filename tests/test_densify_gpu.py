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


def _random_merge_case(seed, n_img=6, n_feat=40, n_match=300, n_points=25):
    from paper_1512_06235_b200.types import Camera, FeatureRef, FeatureSet, Model

    rng = np.random.default_rng(seed)
    ids = sorted(rng.choice(1000, size=n_img, replace=False).tolist())
    sets = {i: FeatureSet(image_id=i, width=100, height=100,
                          xy=np.zeros((n_feat, 2), np.float32), scale=np.ones(n_feat, np.float32),
                          orientation=np.zeros(n_feat, np.float32),
                          descriptors=np.zeros((n_feat, 128), np.uint8)) for i in ids}
    model = Model()
    for i in ids:
        model.attach_camera(Camera(K=np.eye(3), R=np.eye(3), t=np.zeros(3), image_id=i))
    used = set()
    for _ in range(n_points):
        imgs = rng.choice(ids, size=int(rng.integers(2, 4)), replace=False)
        refs = []
        for i in imgs:
            f = int(rng.integers(0, n_feat))
            if (i, f) not in used:
                used.add((int(i), f))
                refs.append(FeatureRef(int(i), f))
        if len({r.image_id for r in refs}) >= 2:
            model.add_point(np.zeros(3), refs)
    q_img, q_fid, t_img, t_fid, dist = [], [], [], [], []
    for _ in range(n_match):
        a, b = rng.choice(ids, size=2, replace=False)
        q_img.append(int(a)); t_img.append(int(b))
        q_fid.append(int(rng.integers(0, n_feat))); t_fid.append(int(rng.integers(0, n_feat)))
        dist.append(float(np.float32(rng.integers(0, 40) * 0.5)))   # ties on purpose
    return sets, model, [np.array(x) for x in (q_img, q_fid, t_img, t_fid)] + [np.array(dist)]


@pytest.mark.parametrize("seed", range(12))
def test_device_track_merge_equals_host_restatement(seed):
    """msfm_merge_tracks against the CPU restatement of densify.py:68-158 on
    random match graphs with owned features, bridges and distance ties."""
    import torch

    from oracle.densify import merge_tracks
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.densify import merge_tracks_device

    sets, model, (qi, qf, ti, tf, d) = _random_merge_case(seed, n_match=[30, 300, 1500][seed % 3])
    want_new, want_ext = merge_tracks(qi, qf, ti, tf, d, model)
    bank = FeatureBank(sets)
    off = {i: int(bank.offsets[bank.index_of[i]]) for i in sets}
    u = torch.tensor([off[i] + f for i, f in zip(qi, qf)], dtype=torch.int32, device=bank.device)
    v = torch.tensor([off[i] + f for i, f in zip(ti, tf)], dtype=torch.int32, device=bank.device)
    dist = torch.tensor(d, dtype=torch.float32, device=bank.device)
    got_new, got_ext = merge_tracks_device(bank, u, v, dist, model)
    assert got_new == [sorted(t) for t in want_new]
    assert {k: sorted(v) for k, v in got_ext.items()} == {k: sorted(v) for k, v in want_ext.items()}
    assert list(got_ext) == list(want_ext)


@pytest.mark.parametrize("seed", range(4))
def test_device_covisibility_equals_host(seed):
    """msfm_covisibility == len(model.covisible_points(a, b)) for every pair."""
    from oracle.densify import covisibility_counts as host_counts
    from paper_1512_06235_b200.densify import covisibility_counts

    _, model, _ = _random_merge_case(seed, n_img=[3, 8, 20, 2][seed], n_points=[5, 60, 300, 0][seed])
    ids = model.image_ids()
    got = covisibility_counts(model, ids)
    want = host_counts(model, ids)
    off = ~np.eye(len(ids), dtype=bool)          # the diagonal is not a pair
    np.testing.assert_array_equal(got[off], want[off])
    for a in ids[:5]:
        for b in ids[:5]:
            if a != b:
                assert got[ids.index(a), ids.index(b)] == len(model.covisible_points(a, b))
