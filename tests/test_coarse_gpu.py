"""Coarse two-view geometry on the device against the reference's
estimate_fundamental_ransac (geometry.py:153-198): inlier masks identical,
F within 1e-6 (entries of the Frobenius-normalized matrix)."""

import os

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu


def test_fransac_equals_reference():
    from paper_1512_06235_b200.fundamental import estimate_fundamental_ransac
    from paper_1512_06235_b200.types import InsufficientDataError

    z = np.load(os.path.join(GOLDEN, "fransac_cases.npz"))
    for k in range(int(z["n_cases"])):
        q, c, seed = z[f"c{k}_q"], z[f"c{k}_c"], int(z[f"c{k}_seed"])
        status = str(z[f"c{k}_status"])
        if status == "insufficient":
            with pytest.raises(InsufficientDataError):
                estimate_fundamental_ransac(q, c, seed=seed)
            continue
        if status == "overflow":
            with pytest.raises(OverflowError):
                estimate_fundamental_ransac(q, c, seed=seed)
            continue
        geom, mask = estimate_fundamental_ransac(q, c, seed=seed)
        np.testing.assert_array_equal(mask, z[f"c{k}_mask"], err_msg=f"case {k}")
        assert geom.inlier_count == int(z[f"c{k}_count"])
        assert geom.degenerate_planar == bool(z[f"c{k}_planar"]), k
        np.testing.assert_allclose(geom.F, z[f"c{k}_F"], atol=1e-6, err_msg=f"case {k}")


@pytest.mark.parametrize("name", ["coarse_graph_holdout.npz", "coarse_graph_c1eta.npz"])
def test_coarse_matchgraph_equals_reference(name):
    """build_coarse_matchgraph (matching.py:208-249): same edges, hybrid match
    lists (ids, f32 distances, ratios), inlier masks; F within 1e-6."""
    import ast

    from paper_1512_06235_b200.coarse import build_coarse_matchgraph, hybrid_match
    from paper_1512_06235_b200.synth import SceneSpec, generate_scene

    z = np.load(os.path.join(GOLDEN, name))
    scene = generate_scene(SceneSpec(**ast.literal_eval(str(z["spec"]))))
    store = scene.store()
    if float(z["eta"]) > 0:
        store.apply_eta(float(z["eta"]))
    ids = sorted(store.sets)
    assert [store.sets[i].coarse_count for i in ids] == z["coarse"].tolist()
    graph = build_coarse_matchgraph(store.sets)
    want = [tuple(e) for e in z["edges"].tolist()]
    assert sorted(graph.edges) == want
    for e, key in enumerate(want):
        ed = graph.edges[key]
        np.testing.assert_array_equal([m.query.feature_id for m in ed.matches], z[f"e{e}_q"])
        np.testing.assert_array_equal([m.target.feature_id for m in ed.matches], z[f"e{e}_t"])
        np.testing.assert_array_equal([m.distance for m in ed.matches], z[f"e{e}_d"])
        np.testing.assert_array_equal([m.ratio for m in ed.matches], z[f"e{e}_r"])
        np.testing.assert_array_equal(ed.inlier_mask, z[f"e{e}_mask"])
        assert ed.geometry.inlier_count == int(z[f"e{e}_count"])
        np.testing.assert_allclose(ed.geometry.F, z[f"e{e}_F"], atol=1e-6)
    # the per-pair drop-in on a few pairs (also ones without an edge)
    for a, b, cnt in z["hybrid_counts"][::7].tolist():
        assert len(hybrid_match(store.sets[a], store.sets[b])) == cnt
