"""The CPU oracle is pinned to the reference's own outputs (golden fixtures)."""

import numpy as np
import pytest

from golden_io import GUIDED_FIXTURES, load, scene_hash
from oracle import guided as og
from paper_1512_06235_b200.geometry import fundamental_from_poses


@pytest.mark.parametrize("name", GUIDED_FIXTURES)
def test_synth_regenerates_fixture_scene(name):
    _, scene, h, _ = load(name)
    assert scene_hash(scene) == h


@pytest.mark.parametrize("name", GUIDED_FIXTURES)
def test_guided_oracle_matches_reference(name):
    _, scene, _, pairs = load(name)
    for p in pairs:
        fq, ft = scene.feature_sets[p["q"]], scene.feature_sets[p["t"]]
        F = fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]]).F
        qi = np.arange(len(fq)) if p["qi"] is None else p["qi"]
        q, t, d, r, st = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                         ft.width, ft.height, F, qi)
        np.testing.assert_array_equal(q, p["mq"])
        np.testing.assert_array_equal(t, p["mt"])
        np.testing.assert_array_equal(d.astype(np.float64), p["dist"])
        np.testing.assert_array_equal(r.astype(np.float64), p["ratio"])
        np.testing.assert_array_equal(st, p["stats"])


def test_oracle_hypot_is_glibc():
    rng = np.random.default_rng(0)
    a = rng.normal(size=20000) * 1e3
    b = rng.normal(size=20000)
    lib = og.lib()
    got = np.array([lib.oracle_hypot(float(x), float(y)) for x, y in zip(a, b)])
    np.testing.assert_array_equal(got, np.hypot(a, b))
