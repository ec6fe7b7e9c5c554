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


@pytest.mark.gpu
def test_device_angle_gate_on_long_narrow_tracks():
    """The widest-ray-angle gate (geometry.py:350-356) around its threshold on long
    tracks (the kernel stops at the first pair that reaches min_angle): statuses,
    points and errors equal to the oracle's full pairwise scan."""
    from paper_1512_06235_b200.triangulation import triangulate_batch

    rng = np.random.default_rng(7)
    C = 240
    ang = np.radians(np.arange(C) * 0.06)                 # 0.06 deg between neighbours
    K = np.tile(np.array([[2600.0, 0, 1536], [0, 2600.0, 1152], [0, 0, 1]]), (C, 1, 1))
    R = np.zeros((C, 3, 3))
    t = np.zeros((C, 3))
    for c in range(C):
        cen = np.array([8 * np.cos(ang[c]), 0.0, 8 * np.sin(ang[c])])
        z = -cen / np.linalg.norm(cen)
        x = np.cross([0, 1.0, 0], z)
        x /= np.linalg.norm(x)
        R[c] = np.stack([x, np.cross(z, x), z])
        t[c] = -R[c] @ cen
    T = 400
    lens = rng.integers(2, 60, size=T)
    ptr = np.zeros(T + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    cam = np.empty(ptr[-1], np.int32)
    pix = np.empty((ptr[-1], 2))
    for k in range(T):
        c0 = int(rng.integers(0, C - lens[k]))
        cs = c0 + rng.permutation(lens[k])               # shuffled view order
        cam[ptr[k]:ptr[k + 1]] = cs
        Xw = rng.normal(size=3) * 0.5
        xc = np.einsum("cij,j->ci", R[cs], Xw) + t[cs]
        uv = np.einsum("cij,cj->ci", K[cs], xc)
        pix[ptr[k]:ptr[k + 1]] = uv[:, :2] / uv[:, 2:3] + rng.normal(size=(lens[k], 2)) * 0.2
    st, X, err = triangulate_batch(K, R, t, ptr, cam, pix)
    code = {"ok": 1, "rejected": 0, "degenerate": -1}
    n_rej = 0
    for k in range(T):
        lo, hi = ptr[k], ptr[k + 1]
        c = cam[lo:hi]
        s, Xo, eo = otri.triangulate(K[c], R[c], t[c], pix[lo:hi])
        assert st[k] == code[s], k
        n_rej += s == "rejected"
        if s == "ok":
            np.testing.assert_allclose(X[k], Xo, rtol=1e-6, atol=1e-9)
            np.testing.assert_allclose(err[k], eo, atol=1e-6)
    assert 0 < n_rej < T                                  # both sides of the gate exercised
