"""The localization oracle is pinned to the reference's outputs."""

import numpy as np
import pytest

from golden_io import GOLDEN, load_localize
from oracle import localize as ol
from paper_1512_06235_b200 import scenes


@pytest.mark.parametrize("name", ["localize_holdout.npz", "localize_c2mini.npz"])
def test_snapshot_and_knn_and_direct_search(name):
    kw, scene, snap, z = load_localize(name)
    assert len(snap.point_xyz) == int(z["n_points"])
    S, n = scenes.track_sums(scene, snap)
    agree = total = 0
    for q in z["queries"]:
        q = int(q)
        F = scene.feature_sets[q].descriptors
        idx, nb, ns = ol.knn2_exact(S, n, F)
        ref_idx = z[f"q{q}_knn_idx"][:, 0]
        agree += int((idx == ref_idx).sum()); total += len(idx)
        corr = ol.direct_3d2d(np.arange(len(S)), S, n, F)
        np.testing.assert_array_equal(corr, z[f"q{q}_corr"])
    # the reference's exact path is float32 (inexact for means); report-level agreement
    assert agree / total > 0.999


def test_pnp_oracle_equals_reference_cases():
    z = np.load(f"{GOLDEN}/pnp_cases.npz")
    for k in range(int(z["n_cases"])):
        X, uv, K, seed = z[f"c{k}_X"], z[f"c{k}_uv"], z[f"c{k}_K"], int(z[f"c{k}_seed"])
        status = str(z[f"c{k}_status"])
        if status == "overflow":
            with pytest.raises(OverflowError):
                ol.pnp_ransac(X, uv, K, seed=seed)
            continue
        res = ol.pnp_ransac(X, uv, K, seed=seed)
        if status == "none":
            assert res is None
            continue
        R, t, mask = res
        np.testing.assert_array_equal(mask, z[f"c{k}_mask"])
        np.testing.assert_allclose(R, z[f"c{k}_R"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(t, z[f"c{k}_t"], rtol=1e-12, atol=1e-12)


def test_pnp_oracle_on_localization_fixtures():
    for name in ["localize_holdout.npz", "localize_c2mini.npz"]:
        kw, scene, snap, z = load_localize(name)
        for q in z["queries"]:
            q = int(q)
            c = z[f"q{q}_corr"]
            status = str(z[f"q{q}_status"])
            if status == "below_gate":
                continue
            X = snap.point_xyz[c[:, 0]]
            uv = scene.feature_sets[q].xy[c[:, 1]].astype(np.float64)
            K = scene.cameras[q].K
            if status == "overflow":
                with pytest.raises(OverflowError):
                    ol.pnp_ransac(X, uv, K, seed=q)
                continue
            R, t, mask = ol.pnp_ransac(X, uv, K, seed=q)
            np.testing.assert_array_equal(mask, z[f"q{q}_mask"])
            np.testing.assert_allclose(R, z[f"q{q}_R"], atol=1e-12)
