"""Triangulation: oracle pinned to the reference fixture (CPU); device kernel vs
reference (GPU): identical accept/reject/degenerate flags, points within 1e-6
relative, reprojection error within 1e-6 px (stated bars: 1e-4 rel, 1e-3 px)."""

import ast

import numpy as np
import pytest

from golden_io import GOLDEN
from oracle import triangulate as otri
from paper_1512_06235_b200.synth import SceneSpec, generate_scene

Z = np.load(f"{GOLDEN}/triangulate.npz")
SCENE = None


def scene():
    global SCENE
    if SCENE is None:
        SCENE = generate_scene(SceneSpec(**ast.literal_eval(str(Z["spec"]))))
    return SCENE


def track_arrays():
    sc = scene()
    ptr, obs = Z["ptr"], Z["obs"]
    K = np.stack([c.K for c in sc.cameras])
    R = np.stack([c.R for c in sc.cameras])
    t = np.stack([c.t for c in sc.cameras])
    pix = np.stack([sc.feature_sets[int(i)].xy[int(f)].astype(np.float64) for i, f in obs])
    return K, R, t, ptr, obs[:, 0], pix


def test_oracle_matches_reference_tracks():
    K, R, t, ptr, cam, pix = track_arrays()
    for k in range(0, int(Z["n_tracks"]), 7):
        lo, hi = ptr[k], ptr[k + 1]
        c = cam[lo:hi]
        s, X, e = otri.triangulate(K[c], R[c], t[c], pix[lo:hi])
        assert s == str(Z["status"][k])
        if s == "ok":
            np.testing.assert_allclose(X, Z["X"][k], rtol=1e-12, atol=1e-12)


def test_oracle_edge_cases():
    for k in range(int(Z["n_edges"])):
        s, X, e = otri.triangulate(Z[f"e{k}_K"], Z[f"e{k}_R"], Z[f"e{k}_t"], Z[f"e{k}_pix"])
        assert s == str(Z[f"e{k}_status"]), k


@pytest.mark.gpu
def test_device_batch_matches_reference():
    from paper_1512_06235_b200.triangulation import triangulate_batch

    K, R, t, ptr, cam, pix = track_arrays()
    st, X, err = triangulate_batch(K, R, t, ptr, cam, pix)
    want = np.array([{"ok": 1, "rejected": 0, "degenerate": -1}[str(s)] for s in Z["status"]])
    np.testing.assert_array_equal(st, want)
    ok = want == 1
    np.testing.assert_allclose(X[ok], Z["X"][ok], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(err[ok], Z["err"][ok], atol=1e-6)


@pytest.mark.gpu
def test_device_dropin_edge_cases():
    from paper_1512_06235_b200.triangulation import triangulate_track
    from paper_1512_06235_b200.types import Camera, DegenerateGeometryError, InsufficientDataError

    for k in range(int(Z["n_edges"])):
        obs = [(Camera(K=Kc, R=Rc, t=tc, image_id=i), p) for i, (Kc, Rc, tc, p) in
               enumerate(zip(Z[f"e{k}_K"], Z[f"e{k}_R"], Z[f"e{k}_t"], Z[f"e{k}_pix"]))]
        s = str(Z[f"e{k}_status"])
        if s == "degenerate":
            with pytest.raises(DegenerateGeometryError):
                triangulate_track(obs)
        elif s == "rejected":
            assert triangulate_track(obs) is None
        else:
            r = triangulate_track(obs)
            np.testing.assert_allclose(r.point, Z[f"e{k}_X"], rtol=1e-6, atol=1e-9)
            assert abs(r.mean_error - float(Z[f"e{k}_err"])) < 1e-6
    with pytest.raises(InsufficientDataError):
        triangulate_track(obs[:1])
