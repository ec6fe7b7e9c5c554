"""2-NN drop-ins (descriptors.py:35-139) against the reference's own outputs
(tests/golden/descriptors_knn2.npz, made by make_golden_descriptors.py)."""

import os

import numpy as np
import pytest

from oracle import localize as ol

GOLD = os.path.join(os.path.dirname(__file__), "golden", "descriptors_knn2.npz")


def _cases():
    z = np.load(GOLD)
    for name in z["names"]:
        yield str(name), z[f"{name}_q"], z[f"{name}_t"], z[f"{name}_dist"], z[f"{name}_idx"], \
            z[f"{name}_stats"]


def test_oracle_two_nearest_pinned_to_reference():
    for name, q, t, dist, idx, _ in _cases():
        od, oi = ol.two_nearest(q, t)
        assert np.array_equal(oi, idx), name
        assert np.array_equal(od, dist), name


def test_fixture_has_ties():
    z = np.load(GOLD)
    q, t = z["ties_q"].astype(np.int64), z["ties_t"].astype(np.int64)
    d2 = ((q[:, None, :] - t[None, :, :]) ** 2).sum(-1)
    srt = np.sort(d2, 1)
    # a quarter of the rows tie for the best, a third for the second
    assert (srt[:, 0] == srt[:, 1]).mean() > 0.2 and (srt[:, 1] == srt[:, 2]).mean() > 0.3


def test_non_integer_queries_rejected():
    from paper_1512_06235_b200.descriptors import _as_u8
    with pytest.raises(ValueError):
        _as_u8(np.full((2, 128), 0.5, np.float32), "queries")
    with pytest.raises(ValueError):
        _as_u8(np.full((2, 128), 256.0, np.float32), "queries")
    assert _as_u8(np.zeros((0, 128)), "q").shape == (0, 128)


@pytest.mark.gpu
def test_two_nearest_bruteforce_equals_reference():
    from paper_1512_06235_b200.descriptors import two_nearest_bruteforce
    from paper_1512_06235_b200.types import SearchStats
    for name, q, t, dist, idx, stats in _cases():
        st = SearchStats()
        d, i = two_nearest_bruteforce(q.astype(np.float32), t, st)
        assert np.array_equal(i, idx), name
        assert np.array_equal(d, dist), name
        assert d.dtype == np.float64 and i.dtype == np.int64
        assert (st.queries, st.candidates) == (int(stats[0]), int(stats[1])), name


@pytest.mark.gpu
def test_descriptor_index_equals_reference():
    from paper_1512_06235_b200.descriptors import DescriptorIndex
    from paper_1512_06235_b200.types import SearchStats
    for name, q, t, dist, idx, stats in _cases():
        index = DescriptorIndex(t.astype(np.float32))
        st = SearchStats()
        d, i = index.knn2(q, st)
        assert np.array_equal(i, idx) and np.array_equal(d, dist), name
        assert (st.queries, st.candidates) == (int(stats[2]), int(stats[3])), name
        # reused index, second batch of queries
        d2, i2 = index.knn2(q[::-1])
        assert np.array_equal(i2, idx[::-1]), name


@pytest.mark.gpu
def test_two_nearest_large_against_oracle():
    from paper_1512_06235_b200.descriptors import two_nearest_bruteforce
    rng = np.random.default_rng(3)
    base = rng.integers(0, 256, (300, 128), dtype=np.uint8)
    q = base[rng.integers(0, 300, 3000)]
    t = np.concatenate([base[rng.integers(0, 300, 5000)],
                        rng.integers(0, 256, (9000, 128), dtype=np.uint8)])
    d, i = two_nearest_bruteforce(q, t)
    od, oi = ol.two_nearest(q, t)
    assert np.array_equal(i, oi) and np.array_equal(d, od)
