"""Seeded RANSAC hypothesis sets (host side, C): numpy's
``default_rng(seed).choice(n, 6, replace=False)`` stream, as pnp_ransac draws
it (reconstruct.py:185-194).  Sampling is independent of outcomes, so the whole
stream can be produced up front and scored on the device."""

from __future__ import annotations

import numpy as np

from . import _lib


def rng_state(seed: int):
    """PCG64 state words of np.random.default_rng(seed) (SeedSequence done by numpy)."""
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    words = np.array([s >> 64, s & (2**64 - 1), inc >> 64, inc & (2**64 - 1)], dtype=np.uint64)
    return words, int(st["has_uint32"]), int(st["uinteger"])


def ransac_samples(seed: int, n: int, count: int, sample_size: int = 6) -> np.ndarray:
    """(count, sample_size) int32 — rows are the reference's consecutive samples."""
    lib = _lib.load(require_device=False)
    words, has32, u32 = rng_state(seed)
    out = np.zeros((count, sample_size), dtype=np.int32)
    _lib.check(lib.msfm_ransac_samples(words.ctypes.data, has32, u32, int(n), int(sample_size),
                                       int(count), out.ctypes.data, None), "msfm_ransac_samples")
    return out
