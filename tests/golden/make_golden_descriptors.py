"""Golden fixtures for the 2-NN drop-ins from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_descriptors.py

Runs msfm.descriptors.two_nearest_bruteforce (descriptors.py:35-72) and the
exact DescriptorIndex.knn2 (descriptors.py:105-139) on seeded uint8 inputs: a
random case, a low-entropy case with many equal distances (tie breaking toward
the lower index, first and second column), a single-target case (+inf / -1) and
an empty query set.  Inputs and outputs (dist, idx, SearchStats) are stored.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("MSFM_REF_PATH", "/root/reference/pkg/src"))

from msfm.descriptors import DescriptorIndex, SearchStats, two_nearest_bruteforce  # noqa: E402


def cases():
    rng = np.random.default_rng(2024)
    yield "random", rng.integers(0, 256, (700, 128), dtype=np.uint8), \
        rng.integers(0, 256, (1500, 128), dtype=np.uint8)
    yield "ties", rng.integers(0, 2, (600, 128), dtype=np.uint8) * 3, \
        rng.integers(0, 2, (900, 128), dtype=np.uint8) * 3
    base = rng.integers(0, 256, (40, 128), dtype=np.uint8)
    yield "duplicates", base[rng.integers(0, 40, 300)], base[rng.integers(0, 40, 500)]
    yield "single", rng.integers(0, 256, (50, 128), dtype=np.uint8), \
        rng.integers(0, 256, (1, 128), dtype=np.uint8)
    yield "empty", np.zeros((0, 128), np.uint8), rng.integers(0, 256, (30, 128), dtype=np.uint8)
    yield "extreme", np.where(rng.random((300, 128)) < 0.5, 0, 255).astype(np.uint8), \
        np.where(rng.random((2000, 128)) < 0.5, 0, 255).astype(np.uint8)


def main():
    out = {}
    for name, q, t in cases():
        st = SearchStats()
        dist, idx = two_nearest_bruteforce(q, t, st)
        ist = SearchStats()
        idist, iidx = DescriptorIndex(t.astype(np.float32)).knn2(q.astype(np.float32), ist)
        assert np.array_equal(dist, idist) and np.array_equal(idx, iidx)
        out[f"{name}_q"] = q
        out[f"{name}_t"] = t
        out[f"{name}_dist"] = dist
        out[f"{name}_idx"] = idx
        out[f"{name}_stats"] = np.array([st.queries, st.candidates, ist.queries, ist.candidates])
    out["names"] = np.array([n for n, _, _ in cases()])
    np.savez_compressed(os.path.join(HERE, "descriptors_knn2.npz"), **out)
    print("wrote descriptors_knn2.npz:", list(out["names"]))


if __name__ == "__main__":
    main()
