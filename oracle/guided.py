"""ctypes wrapper of liboracle.so: ``oracle_guided_match`` restates
``msfm.guided.guided_match_pair`` (pkg/src/msfm/guided.py:393-480) in C.

ORACLE — test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.oracle_guided_match.restype = ctypes.c_int
        L.oracle_guided_match.argtypes = [P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_float, ctypes.c_float, P, P, P, P, ctypes.c_int, P]
        L.oracle_hypot.restype = ctypes.c_double
        L.oracle_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def guided_match(qxy, qdesc, txy, tdesc, width, height, F, query_indices, *,
                 d=8.0, inflation=1.25, grid_d=None, ratio=0.8, single_cap=45.0):
    """Returns (q, t, dist f32, ratio f32, stats[2]) sorted by q."""
    qxy = np.ascontiguousarray(qxy, np.float32); txy = np.ascontiguousarray(txy, np.float32)
    qdesc = np.ascontiguousarray(qdesc, np.uint8); tdesc = np.ascontiguousarray(tdesc, np.uint8)
    F = np.ascontiguousarray(F, np.float64).reshape(9)
    qi = np.ascontiguousarray(query_indices, np.int32)
    cap = max(1, len(qi))
    oq = np.zeros(cap, np.int32); ot = np.zeros(cap, np.int32)
    od = np.zeros(cap, np.float32); orr = np.zeros(cap, np.float32)
    stats = np.zeros(2, np.int64)
    D = grid_d if grid_d is not None else d * inflation
    n = lib().oracle_guided_match(_p(qxy), _p(qdesc), _p(txy), _p(tdesc), len(txy),
                                  float(width), float(height), _p(F), _p(qi), len(qi),
                                  float(d), float(D), float(ratio), float(single_cap),
                                  _p(oq), _p(ot), _p(od), _p(orr), cap, _p(stats))
    if n < 0:
        raise RuntimeError("oracle output capacity exceeded")
    return oq[:n].copy(), ot[:n].copy(), od[:n].copy(), orr[:n].copy(), stats
