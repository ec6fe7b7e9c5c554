"""The C-ABI library loads and exports every symbol include/msfm_b200.h declares."""

import ctypes
import os
import re

import pytest

from paper_1512_06235_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "msfm_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(msfm_[a-z0-9_]+)\s*\(", src)))


def test_library_exists_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    lib = _lib.load(require_device=False)
    assert lib.msfm_version() >= 1


@pytest.mark.parametrize("name", declared_symbols())
def test_header_symbol_exported(name):
    lib = ctypes.CDLL(_lib.LIB_PATH)
    assert hasattr(lib, name)


def test_binding_covers_header():
    assert set(declared_symbols()) <= set(_lib.EXPORTED)


def test_host_only_entry_points_without_gpu():
    lib = _lib.load(require_device=False)
    buf = (ctypes.c_int32 * 2)()
    assert lib.msfm_grid_dims(3072, 2304, 10.0, buf) == 0
    assert (buf[0], buf[1]) == (308, 231)
    assert lib.msfm_grid_dims(10, 10, 0.0, buf) == -1
    assert b"positive" in lib.msfm_last_error()
    assert lib.msfm_grid_workspace_bytes(1000) > 0


def test_argument_validation_without_gpu():
    """Entry points reject bad arguments with MSFM_EINVAL and a message before any
    device work (no GPU needed)."""
    lib = _lib.load(require_device=False)
    bank = _lib.Bank(None, None, None, None, None, None, 4, 1000)
    # image range outside the bank / inverted
    assert lib.msfm_grid_build_range(ctypes.byref(bank), None, None, None, 100, 3, 2, 0, 10, 0,
                                     10.0, None, None, None, None, None, None, None, None,
                                     10**6, None) == -1
    assert b"images [3, 2)" in lib.msfm_last_error()
    assert lib.msfm_grid_build_range(ctypes.byref(bank), None, None, None, 100, 0, 9, 0, 10, 0,
                                     10.0, None, None, None, None, None, None, None, None,
                                     10**6, None) == -1
    # chunk bounds: host-only planning
    prm = _lib.MatchParams(8.0, 0.8, 45.0, 100, 3, 0, 2)
    import numpy as np
    qoff = np.array([0, 10, 20, 30, 40, 50, 60, 70], np.int64)
    out = np.zeros(10, np.int32)
    nc = lib.msfm_guided_chunk_bounds(7, qoff.ctypes.data, ctypes.byref(prm), out.ctypes.data, 10)
    assert nc == 3 and out[:4].tolist() == [0, 2, 5, 7]      # first chunk 2 pairs, then 3
    # sampler: bad sample size, negative items
    assert lib.msfm_ransac_samples_seeded_device(1, None, None, 0, 4, None, None, None, None) == -1
    assert lib.msfm_ransac_samples_seeded(-1, None, None, 6, 4, None, None) == -1
    # gather / triangulation / pack with negative sizes
    assert lib.msfm_gather_3d2d(None, None, 128, -1, None, None, None, None, None, None, None,
                                None) == -1
    assert lib.msfm_triangulate_batch(None, None, None, -1, None, None, None, 4.0, 1.0, None,
                                      None, None, None) == -1
    assert lib.msfm_pack_matches(-1, None, None, None, None, None, None, None, None, None) == -1
    # zero-sized work is a no-op success
    assert lib.msfm_gather_3d2d(None, None, 128, 0, None, None, None, None, None, None, None,
                                None) == 0
