"""The native hypothesis generator reproduces numpy's Generator.choice stream."""

import numpy as np
import pytest

from paper_1512_06235_b200.sampling import ransac_samples


@pytest.mark.parametrize("seed,n", [(0, 6), (1, 7), (5, 40), (17, 1500), (123, 6000), (99, 9999),
                                    (7, 10000), (3, 65535), (11, 2**20)])
def test_matches_numpy_choice(seed, n):
    if n > 10000:
        pytest.skip("tail-shuffle branch not needed for pnp populations")
    count = 300
    rng = np.random.default_rng(seed)
    ref = np.stack([rng.choice(n, size=6, replace=False) for _ in range(count)])
    np.testing.assert_array_equal(ransac_samples(seed, n, count), ref)


def test_many_seeds_small_populations():
    for seed in range(200):
        n = 6 + seed * 37 % 3000
        rng = np.random.default_rng(seed)
        ref = np.stack([rng.choice(n, size=6, replace=False) for _ in range(20)])
        np.testing.assert_array_equal(ransac_samples(seed, n, 20), ref)


def test_rejects_bad_population():
    with pytest.raises(ValueError):
        ransac_samples(0, 5, 3)


def test_stream_continuation():
    """state_out continues the stream exactly (used for a second RANSAC round)."""
    from paper_1512_06235_b200 import _lib
    from paper_1512_06235_b200.sampling import rng_state

    lib = _lib.load(require_device=False)
    seed, n = 42, 777
    words, has32, u32 = rng_state(seed)
    a = np.zeros((10, 6), np.int32)
    st = np.zeros(6, np.uint64)
    _lib.check(lib.msfm_ransac_samples(words.ctypes.data, has32, u32, n, 6, 10, a.ctypes.data,
                                       st.ctypes.data), "s")
    b = np.zeros((15, 6), np.int32)
    w2 = np.ascontiguousarray(st[:4])
    _lib.check(lib.msfm_ransac_samples(w2.ctypes.data, int(st[4]), int(st[5]), n, 6, 15,
                                       b.ctypes.data, None), "s")
    rng = np.random.default_rng(seed)
    ref = np.stack([rng.choice(n, 6, replace=False) for _ in range(25)])
    np.testing.assert_array_equal(np.vstack([a, b]), ref)


def test_seedsequence_restatement_matches_numpy():
    """msfm_rng_seed_state == np.random.default_rng(seed).bit_generator.state."""
    from paper_1512_06235_b200 import _lib
    from paper_1512_06235_b200.sampling import rng_state

    lib = _lib.load(require_device=False)
    seeds = list(range(0, 300)) + [2**32 - 1, 2**32, 2**32 + 5, 123456789012, 2**63 + 11,
                                   2**64 - 1, 100003 * 19 + 18, 31337]
    out = np.zeros(6, np.uint64)
    for seed in seeds:
        words, has32, u32 = rng_state(seed)
        assert lib.msfm_rng_seed_state(seed, out.ctypes.data) == 0
        np.testing.assert_array_equal(out[:4], words, err_msg=str(seed))
        assert has32 == 0 and u32 == 0


@pytest.mark.parametrize("size", [6, 8])
def test_batched_seeded_samples(size):
    from paper_1512_06235_b200 import _lib

    lib = _lib.load(require_device=False)
    seeds = np.array([3, 1000, 100003 * 4 + 9, 7], np.uint64)
    n = np.array([50, 8, 3000, 123], np.int64)
    count = 40
    out = np.zeros((len(seeds), count, size), np.int32)
    st = np.zeros((len(seeds), 6), np.uint64)
    assert lib.msfm_ransac_samples_seeded(len(seeds), seeds.ctypes.data, n.ctypes.data, size,
                                          count, out.ctypes.data, st.ctypes.data) == 0
    for i in range(len(seeds)):
        rng = np.random.default_rng(int(seeds[i]))
        ref = np.stack([rng.choice(int(n[i]), size=size, replace=False) for _ in range(count)])
        np.testing.assert_array_equal(out[i], ref)
        s = rng.bit_generator.state
        assert int(st[i, 0]) == s["state"]["state"] >> 64
        assert int(st[i, 4]) == s["has_uint32"]


def test_record_replay_equals_loop_replay():
    """The record-only replay of the RANSAC stopping rule equals the literal loop
    (reconstruct.py:190-211 / geometry.py:176-191), OverflowError included."""
    from paper_1512_06235_b200.pnp import _replay, _replay_records

    rng = np.random.default_rng(0)
    for _ in range(3000):
        H = int(rng.choice([8, 64, 256, 2048]))
        n = int(rng.integers(6, 3000))
        mode = int(rng.integers(0, 3))
        if mode == 0:
            c = rng.integers(-1, n + 1, size=H)
        elif mode == 1:
            c = rng.integers(0, max(2, n // 50), size=H)
        else:
            c = np.sort(rng.integers(-1, n + 1, size=H))
        ev = int(rng.integers(1, H + 1))
        power = int(rng.choice([6, 8]))
        out = []
        for f in (_replay, _replay_records):
            try:
                out.append(f(c, ev, n, H, 0.999, power))
            except OverflowError:
                out.append("overflow")
        assert out[0] == out[1]


def test_batched_replay_equals_loop_replay():
    from paper_1512_06235_b200.pnp import _replay, _replay_batch

    rng = np.random.default_rng(1)
    for _ in range(60):
        A, H = int(rng.integers(1, 40)), int(rng.choice([64, 256, 2048]))
        n = rng.integers(6, 3000, size=A)
        C = np.where(rng.random((A, H)) < 0.5, rng.integers(-1, 5, size=(A, H)),
                     rng.integers(-1, 3000, size=(A, H)))
        C = np.minimum(C, n[:, None])
        ev = int(rng.integers(1, H + 1))
        power = int(rng.choice([6, 8]))
        got = _replay_batch(C, ev, n, H, 0.999, power)
        for k in range(A):
            try:
                want = _replay(C[k], ev, int(n[k]), H, 0.999, power)
            except OverflowError:
                want = "overflow"
            assert got[k] == want
