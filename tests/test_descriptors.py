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


def test_non_integer_rows_take_the_real_valued_path():
    from paper_1512_06235_b200.descriptors import _as_u8
    assert _as_u8(np.full((2, 128), 0.5, np.float32)) is None
    assert _as_u8(np.full((2, 128), 256.0, np.float32)) is None
    assert _as_u8(np.full((2, 64), 3.0, np.float32)) is None
    assert _as_u8(np.zeros((0, 128))).shape == (0, 128)
    assert _as_u8(np.full((3, 128), 7.0)).dtype == np.uint8


@pytest.mark.gpu
def test_float_rows_equal_f64_brute_force():
    """Arbitrary float32 rows (test_matching.py:54-71 style: normal draws, noisy
    integers, exact duplicates for ties, a single target): indices equal a numpy
    f64 brute force with lowest-index ties; distances its sqrt."""
    from paper_1512_06235_b200.descriptors import DescriptorIndex, two_nearest_bruteforce

    rng = np.random.default_rng(11)
    t = rng.normal(size=(700, 128)).astype(np.float32)
    t[5] = t[3]                                  # a tie at the same distance
    q = rng.normal(size=(60, 128)).astype(np.float32)
    q[0] = t[3]
    for qq, tt in [(q, t), (t[:50] + rng.normal(0, 4, (50, 128)).astype(np.float32), t),
                   (q[:5], t[:1])]:
        d, i = two_nearest_bruteforce(qq, tt)
        D = ((qq[:, None, :].astype(np.float64) - tt[None, :, :].astype(np.float64)) ** 2).sum(-1)
        o = np.argsort(D, axis=1, kind="stable")
        assert (i[:, 0] == o[:, 0]).all()
        if len(tt) > 1:
            assert (i[:, 1] == o[:, 1]).all()
            np.testing.assert_allclose(d[:, 1], np.sqrt(D[np.arange(len(qq)), o[:, 1]]), rtol=1e-12)
        else:
            assert (i[:, 1] == -1).all() and np.isinf(d[:, 1]).all()
        np.testing.assert_allclose(d[:, 0], np.sqrt(D[np.arange(len(qq)), o[:, 0]]), rtol=1e-12)
    assert two_nearest_bruteforce(q, t)[1][0, 0] == 3
    idx = DescriptorIndex(t, exact_threshold=100, leaf_size=4, max_leaf_visits=4)
    assert not idx.exact                          # the reference would take its kd-tree here
    np.testing.assert_array_equal(idx.knn2(q)[1], two_nearest_bruteforce(q, t)[1])


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
