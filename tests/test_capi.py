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
