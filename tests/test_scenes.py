"""Workload recipes reproduce the reference densify inputs (pairs, roles, untracked)."""

import numpy as np

from golden_io import load
from paper_1512_06235_b200 import scenes


def test_c1_pair_workload_matches_reference_densify():
    _, scene, _, pairs = load("guided_C1.npz")
    snap = scenes.coarse_snapshot(scene, range(20))
    wl = scenes.pair_workload(scene, snap)
    assert len(wl.pairs) == len(pairs)
    for k, p in enumerate(pairs):
        assert (wl.q_img[k], wl.t_img[k]) == (p["q"], p["t"])
        np.testing.assert_array_equal(wl.untracked[p["q"]], p["qi"])


def test_8k_pair_workload_matches_reference_densify():
    _, scene, _, pairs = load("guided_8k.npz")
    snap = scenes.coarse_snapshot(scene, range(10))
    wl = scenes.pair_workload(scene, snap)
    for k, p in enumerate(pairs):
        assert (wl.q_img[k], wl.t_img[k]) == (p["q"], p["t"])
        np.testing.assert_array_equal(wl.untracked[p["q"]], p["qi"])
