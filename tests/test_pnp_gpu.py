"""GPU PnP-RANSAC vs the reference's outputs: identical inlier masks, poses within tolerance."""

import numpy as np
import pytest

from golden_io import GOLDEN, load_localize

pytestmark = pytest.mark.gpu

R_TOL = 1e-6     # stated tolerance (relative/absolute on rotation entries); expected ~1e-10
T_TOL = 1e-6


def _check(res, R, t, mask):
    assert res is not None
    gR, gt, gm = res
    np.testing.assert_array_equal(gm, mask)
    np.testing.assert_allclose(gR, R, atol=R_TOL)
    np.testing.assert_allclose(gt, t, rtol=T_TOL, atol=T_TOL)


def test_pnp_cases_match_reference():
    from paper_1512_06235_b200.pnp import pnp_ransac

    z = np.load(f"{GOLDEN}/pnp_cases.npz")
    for k in range(int(z["n_cases"])):
        X, uv, K, seed = z[f"c{k}_X"], z[f"c{k}_uv"], z[f"c{k}_K"], int(z[f"c{k}_seed"])
        status = str(z[f"c{k}_status"])
        if status == "overflow":
            with pytest.raises(OverflowError):
                pnp_ransac(X, uv, K, seed=seed)
        elif status == "none":
            assert pnp_ransac(X, uv, K, seed=seed) is None
        else:
            _check(pnp_ransac(X, uv, K, seed=seed), z[f"c{k}_R"], z[f"c{k}_t"], z[f"c{k}_mask"])


@pytest.mark.parametrize("name", ["localize_holdout.npz", "localize_c2mini.npz"])
def test_batched_pnp_on_reference_correspondences(name):
    from paper_1512_06235_b200.pnp import pnp_batch

    kw, scene, snap, z = load_localize(name)
    qs = [int(q) for q in z["queries"] if str(z[f"q{int(q)}_status"]) != "below_gate"]
    X = [snap.point_xyz[z[f"q{q}_corr"][:, 0]] for q in qs]
    uv = [scene.feature_sets[q].xy[z[f"q{q}_corr"][:, 1]].astype(np.float64) for q in qs]
    K = [scene.cameras[q].K for q in qs]
    res = pnp_batch(X, uv, K, qs)
    for q, r in zip(qs, res):
        status = str(z[f"q{q}_status"])
        assert r.status == status, (q, r.status, status)
        if status == "ok":
            _check((r.R, r.t, r.mask), z[f"q{q}_R"], z[f"q{q}_t"], z[f"q{q}_mask"])


def test_insufficient_raises():
    from paper_1512_06235_b200.pnp import pnp_ransac
    from paper_1512_06235_b200.types import InsufficientDataError

    with pytest.raises(InsufficientDataError):
        pnp_ransac(np.zeros((5, 3)), np.zeros((5, 2)), np.eye(3))


def test_flat_batch_equals_list_batch():
    """pnp_batch_flat (concatenated correspondences) == pnp_batch (lists), incl.
    images under the 6-correspondence floor."""
    import os

    from golden_io import GOLDEN
    from paper_1512_06235_b200.pnp import pnp_batch, pnp_batch_flat

    z = np.load(os.path.join(GOLDEN, "pnp_cases.npz"))
    ks = list(range(int(z["n_cases"])))
    X = [z[f"c{k}_X"] for k in ks] + [z["c0_X"][:4]]
    uv = [z[f"c{k}_uv"] for k in ks] + [z["c0_uv"][:4]]
    K = [z[f"c{k}_K"] for k in ks] + [z["c0_K"]]
    seeds = [int(z[f"c{k}_seed"]) for k in ks] + [1]
    a = pnp_batch(X, uv, K, seeds)
    off = np.zeros(len(X) + 1, np.int64)
    np.cumsum([len(x) for x in X], out=off[1:])
    b = pnp_batch_flat(np.concatenate(X), np.concatenate(uv), off, K, seeds)
    for ra, rb in zip(a, b):
        assert ra.status == rb.status
        if ra.status == "ok":
            np.testing.assert_array_equal(ra.mask, rb.mask)
            np.testing.assert_array_equal(ra.R, rb.R)


def test_device_sampler_equals_host_sampler():
    """msfm_ransac_samples_seeded_device: the same draws and end states as the host
    restatement (itself pinned draw-for-draw to numpy in test_sampler.py)."""
    import ctypes

    import torch

    from paper_1512_06235_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(4)
    A, H = 37, 300
    n = rng.integers(6, 20000, size=A).astype(np.int64)
    n[:3] = [6, 7, 10001]
    # huge populations: Lemire's bounded draw rejects often (the sequential fixup path)
    n[3:6] = [2**31 + 7, 3 * 2**30, 2**32 - 3]
    seeds = rng.integers(0, 2**63, size=A, dtype=np.uint64)
    seeds[:2] = [0, 2**64 - 1]
    want = np.zeros((A, H, 6), np.int32)
    wst = np.zeros((A, 6), np.uint64)
    _lib.check(lib.msfm_ransac_samples_seeded(A, seeds.ctypes.data, n.ctypes.data, 6, H,
                                              want.ctypes.data, wst.ctypes.data), "host")
    dev = torch.device("cuda")
    d_out = torch.empty((A, H, 6), dtype=torch.int32, device=dev)
    d_st = torch.empty((A, 6), dtype=torch.int64, device=dev)
    d_bad = torch.zeros(1 + A, dtype=torch.int32, device=dev)
    d_seeds = torch.from_numpy(seeds.view(np.int64)).to(dev)
    d_n = torch.from_numpy(n).to(dev)
    _lib.check(lib.msfm_ransac_samples_seeded_device(A, _lib.ptr(d_seeds), _lib.ptr(d_n), 6, H,
                                                     _lib.ptr(d_out), _lib.ptr(d_st),
                                                     _lib.ptr(d_bad), None), "device")
    assert int(d_bad[0].item()) == 0
    np.testing.assert_array_equal(d_out.cpu().numpy(), want)
    np.testing.assert_array_equal(d_st.cpu().numpy().view(np.uint64), wst)
