"""Host replays of the coarse matcher (CPU): the all-targets hybrid schedule equals
the per-pair one (matching.py:143-187), including the SearchStats totals."""

import numpy as np


def test_hybrid_all_equals_per_pair_hybrid():
    from paper_1512_06235_b200.coarse import _hybrid, _hybrid_all
    from paper_1512_06235_b200.types import SearchStats

    rng = np.random.default_rng(0)
    for trial in range(40):
        S, M = int(rng.integers(1, 12)), int(rng.integers(1, 400))
        n_all = M + int(rng.integers(0, 2000))
        idx = rng.integers(-1, 60, size=(S, M))
        d0 = np.sqrt(rng.integers(0, 4000, size=(S, M)).astype(np.float32)).astype(np.float64)
        d1 = np.where(rng.random((S, M)) < 0.1, np.inf,
                      d0 + rng.random((S, M)) * rng.choice([1.0, 30.0, 80.0]))
        d1[rng.random((S, M)) < 0.05] = 0.0
        tiers = rng.integers(1, 2000, size=S)
        ratio = float(rng.choice([0.6, 0.8, 0.95]))
        early = int(rng.choice([4, 16, 64, 10**6]))
        cont = int(rng.choice([0, 4, 20]))
        st_all, st_one = SearchStats(), SearchStats()
        got = _hybrid_all(idx, d0, d1, n_all, M, ratio, 0.1, cont, early, 45.0, tiers, st_all)
        for s in range(S):
            want = _hybrid(idx[s], d0[s], d1[s], n_all, M, ratio, 0.1, cont, early, 45.0,
                           int(tiers[s]), st_one)
            for g, w in zip(got[s], want):
                np.testing.assert_array_equal(g, w)
        assert (st_all.queries, st_all.candidates) == (st_one.queries, st_one.candidates)
