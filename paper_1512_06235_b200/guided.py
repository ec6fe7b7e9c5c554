"""Geometry-aware pair matching: batched device API + reference-shaped drop-in.

``match_pairs`` is the throughput API (one C-ABI call for a whole stage's
pairs, results stay on the device).  ``guided_match_pair`` keeps the exact
signature, defaults, errors and return type of the reference
``msfm.guided.guided_match_pair`` (pkg/src/msfm/guided.py:393-480) and runs the
same kernels on a two-image bank.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bank import FeatureBank
from .types import FeatureRef, Match, SearchStats

BAND_D_PX = 8.0          # guided.py:39
GRID_INFLATION = 1.25    # guided.py:40
RATIO_GUIDED = 0.8       # matching.py:22
SINGLE_CANDIDATE_CAP = 45.0  # matching.py:27
STRATEGIES = {"grid": 0, "linear": 1, "radial": 2}   # guided.py:425-431


# one packed match row (msfm_pack_matches): 16 bytes, little-endian
MATCH_ROW = np.dtype([("pair", "<i4"), ("q", "<u2"), ("t", "<u2"), ("dist", "<f4"), ("ratio", "<f4")])


@dataclass
class PairMatches:
    """Device-resident output of ``match_pairs`` (per-pair segments)."""

    q: "object"       # int32 (total_queries,) — segment k at [qoff[k], qoff[k]+count[k])
    t: "object"
    dist: "object"    # float32
    ratio: "object"   # float32
    count: "object"   # int32 (n_pairs,)
    qoff: np.ndarray  # host int64 (n_pairs+1,)
    stats: "object"   # int64 (n_pairs, 2) or None

    def packed(self, stream=None):
        """Device (rows int32 (total, 4), total): contiguous 16-B match rows in pair order
        (pair, q | t << 16, dist bits, ratio bits), packed on the device."""
        import torch

        lib = _lib.load()
        P = self.count.numel()
        dev = self.q.device
        off = torch.empty(P + 1, dtype=torch.int64, device=dev)
        rows = torch.empty((max(self.q.numel(), 1), 4), dtype=torch.int32, device=dev)
        _lib.check(lib.msfm_pack_matches(P, _lib.ptr(self._qoff_d), _lib.ptr(self.count),
                                         _lib.ptr(self.q), _lib.ptr(self.t), _lib.ptr(self.dist),
                                         _lib.ptr(self.ratio), _lib.ptr(off), _lib.ptr(rows),
                                         _lib.stream_handle(stream)), "msfm_pack_matches")
        total = int(off[P].item())
        return rows[:total], total

    def rows_host(self, pinned=None):
        """Host structured array (MATCH_ROW: pair, q, t, dist, ratio) in pair order:
        one device-side pack and one D2H copy.  With ``pinned`` (int32 (>=total, 4),
        pinned) the result is a zero-copy view of that buffer."""
        import torch

        if self.count.numel() == 0:
            return np.zeros(0, MATCH_ROW)
        rows, total = self.packed()
        if pinned is None or pinned.shape[0] < total:
            pinned = torch.empty((max(total, 1), 4), dtype=torch.int32, pin_memory=True)
        host = pinned[:total]
        host.copy_(rows, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return host.numpy().view(MATCH_ROW).reshape(total)

    def to_host(self, pinned=None):
        """Concatenated (pair_index, q, t, dist, ratio) numpy arrays in pair order."""
        r = self.rows_host(pinned)
        return (r["pair"].astype(np.int64), r["q"].astype(np.int32), r["t"].astype(np.int32),
                r["dist"].copy(), r["ratio"].copy())


def match_pairs(bank: FeatureBank, q_img, t_img, F, query_lists, *, d: float = BAND_D_PX,
                ratio: float = RATIO_GUIDED, inflation: float = GRID_INFLATION,
                grid_d: float | None = None, single_cap: float = SINGLE_CANDIDATE_CAP,
                with_stats: bool = False, chunk_pairs: int = 0, stream=None,
                device_inputs=None, strategy: str = "grid") -> PairMatches:
    """Match every pair k: query image q_img[k] against target t_img[k].

    ``F`` is (P,3,3) float64 (NaN rows mark degenerate pairs, skipped as
    densify.py:161-165 does); ``query_lists[k]`` are the query feature ids
    (ascending, unique).  Image ids are the bank's.
    """
    import torch

    lib = _lib.load()
    if d <= 0:
        raise ValueError(f"cell half-size d must be positive, got {d}")
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    D = float(grid_d) if grid_d is not None else float(d) * float(inflation)
    P = len(q_img)
    dev = bank.device
    if device_inputs is None:
        device_inputs = prepare_pairs(bank, q_img, t_img, F, query_lists)
    pq, pt, pF, qoff_d, qlist_d, qoff = device_inputs[:6]
    qsrc_d = device_inputs[6] if len(device_inputs) > 6 else None
    nq_total = int(qoff[-1]) if P else 0
    grid = bank.grid(D, stream)
    prm = _lib.MatchParams(float(d), float(np.float32(ratio)), float(np.float32(single_cap)),
                           max(bank.max_n, 1), int(chunk_pairs), STRATEGIES[strategy])
    qoff_c = np.ascontiguousarray(qoff, dtype=np.int64)
    ws_bytes = lib.msfm_guided_workspace_bytes(P, qoff_c.ctypes.data, ctypes.byref(prm))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    cap = max(nq_total, 1)
    out_q = torch.empty(cap, dtype=torch.int32, device=dev)
    out_t = torch.empty(cap, dtype=torch.int32, device=dev)
    out_d = torch.empty(cap, dtype=torch.float32, device=dev)
    out_r = torch.empty(cap, dtype=torch.float32, device=dev)
    out_c = torch.zeros(max(P, 1), dtype=torch.int32, device=dev)
    stats = torch.zeros((max(P, 1), 2), dtype=torch.int64, device=dev) if with_stats else None
    b, g = bank.cstruct(), grid.cstruct()
    _lib.check(lib.msfm_guided_match(ctypes.byref(b), ctypes.byref(g), P, _lib.ptr(pq), _lib.ptr(pt),
                                     _lib.ptr(pF), _lib.ptr(qoff_d), _lib.ptr(qlist_d),
                                     _lib.ptr(qsrc_d), qoff_c.ctypes.data, ctypes.byref(prm), _lib.ptr(out_q),
                                     _lib.ptr(out_t), _lib.ptr(out_d), _lib.ptr(out_r),
                                     _lib.ptr(out_c), _lib.ptr(stats), _lib.ptr(ws), ws_bytes,
                                     _lib.stream_handle(stream)),
               "msfm_guided_match")
    res = PairMatches(out_q, out_t, out_d, out_r, out_c[:P], qoff, stats)
    res._qoff_d = qoff_d
    res._keep = (ws, device_inputs)
    return res


def match_pairs_rows(bank: FeatureBank, q_img, t_img, F, query_lists, *, d: float = BAND_D_PX,
                     ratio: float = RATIO_GUIDED, inflation: float = GRID_INFLATION,
                     grid_d: float | None = None, single_cap: float = SINGLE_CANDIDATE_CAP,
                     chunk_pairs: int = 0, stream=None, device_inputs=None,
                     strategy: str = "grid", pinned=None):
    """``match_pairs`` + packing + one pinned host copy per internal chunk, the
    copy of chunk c overlapping the compute of chunk c+1 (msfm_guided_match_rows).
    Returns the host rows as a MATCH_ROW structured array (a view of ``pinned``
    when given: int32 (>= total queries, 4), pinned)."""
    import torch

    lib = _lib.load()
    if d <= 0:
        raise ValueError(f"cell half-size d must be positive, got {d}")
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    D = float(grid_d) if grid_d is not None else float(d) * float(inflation)
    P = len(q_img)
    dev = bank.device
    if device_inputs is None:
        device_inputs = prepare_pairs(bank, q_img, t_img, F, query_lists)
    pq, pt, pF, qoff_d, qlist_d, qoff = device_inputs[:6]
    qsrc_d = device_inputs[6] if len(device_inputs) > 6 else None
    nq_total = int(qoff[-1]) if P else 0
    if P == 0:
        return np.zeros(0, MATCH_ROW)
    grid = bank.grid(D, stream)
    prm = _lib.MatchParams(float(d), float(np.float32(ratio)), float(np.float32(single_cap)),
                           max(bank.max_n, 1), int(chunk_pairs), STRATEGIES[strategy])
    qoff_c = np.ascontiguousarray(qoff, dtype=np.int64)
    ws_bytes = lib.msfm_guided_workspace_bytes(P, qoff_c.ctypes.data, ctypes.byref(prm))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    cap = max(nq_total, 1)
    out_q = torch.empty(cap, dtype=torch.int32, device=dev)
    out_t = torch.empty(cap, dtype=torch.int32, device=dev)
    out_d = torch.empty(cap, dtype=torch.float32, device=dev)
    out_r = torch.empty(cap, dtype=torch.float32, device=dev)
    out_c = torch.zeros(P, dtype=torch.int32, device=dev)
    out_off = torch.empty(P + 1, dtype=torch.int64, device=dev)
    d_rows = torch.empty((cap, 4), dtype=torch.int32, device=dev)
    d_meta = torch.zeros(2 * (P + 1), dtype=torch.int64, device=dev)
    h_meta = torch.zeros(2 * (P + 1), dtype=torch.int64, pin_memory=True)
    if pinned is None or pinned.shape[0] < cap:
        pinned = torch.empty((cap, 4), dtype=torch.int32, pin_memory=True)
    total = ctypes.c_int64(0)
    copy_stream = torch.cuda.Stream(device=dev)
    b, g = bank.cstruct(), grid.cstruct()
    _lib.check(lib.msfm_guided_match_rows(ctypes.byref(b), ctypes.byref(g), P, _lib.ptr(pq),
                                          _lib.ptr(pt), _lib.ptr(pF), _lib.ptr(qoff_d),
                                          _lib.ptr(qlist_d), _lib.ptr(qsrc_d), qoff_c.ctypes.data,
                                          ctypes.byref(prm), _lib.ptr(out_q), _lib.ptr(out_t),
                                          _lib.ptr(out_d), _lib.ptr(out_r), _lib.ptr(out_c),
                                          _lib.ptr(out_off), _lib.ptr(d_rows), _lib.ptr(d_meta),
                                          h_meta.data_ptr(), pinned.data_ptr(), ctypes.byref(total),
                                          _lib.ptr(ws), ws_bytes, _lib.stream_handle(stream),
                                          copy_stream.cuda_stream), "msfm_guided_match_rows")
    n = int(total.value)
    return pinned[:n].numpy().view(MATCH_ROW).reshape(n)


def prepare_pairs(bank: FeatureBank, q_img, t_img, F, query_lists):
    """Stage the pair table on the device (index translation + one copy per array).

    Query lists passed as the same object for several pairs (every pair of one
    query image, densify.py:150-158) are uploaded once and shared."""
    import torch

    P = len(q_img)
    qi = np.array([bank.index_of[int(i)] for i in q_img], dtype=np.int32)
    ti = np.array([bank.index_of[int(i)] for i in t_img], dtype=np.int32)
    Fh = np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(P, 9))
    lens = np.array([len(x) for x in query_lists], dtype=np.int64)
    qoff = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(lens, out=qoff[1:])
    uniq, src = {}, np.zeros(max(P, 1), dtype=np.int64)
    parts, n = [], 0
    for k, x in enumerate(query_lists):
        s = uniq.get(id(x))
        if s is None:
            s = uniq[id(x)] = n
            parts.append(np.asarray(x, dtype=np.int32))
            n += len(x)
        src[k] = s
    qlist = np.concatenate(parts) if n else np.zeros(1, np.int32)
    dev = bank.device

    def up(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)

    return (up(qi), up(ti), up(Fh), up(qoff), up(qlist), qoff, up(src))

# ---------------------------------------------------------------------------
# drop-in for msfm.guided.guided_match_pair
# ---------------------------------------------------------------------------

_BANK_CACHE: dict = {}
_DROPIN_LOCK = threading.Lock()   # densify.py:232-236 may call from a thread pool


def _pair_bank(query_fs, target_fs):
    """Two-image bank, cached by object identity (FeatureSets are immutable
    after load)."""
    key = (id(query_fs), id(target_fs))
    hit = _BANK_CACHE.get(key)
    if hit is not None and hit[0] is query_fs and hit[1] is target_fs:
        return hit[2]
    if len(_BANK_CACHE) > 64:
        _BANK_CACHE.clear()
    bank = FeatureBank({0: query_fs, 1: target_fs})
    _BANK_CACHE[key] = (query_fs, target_fs, bank)
    return bank


class _Sub:
    """Target subset view (target_indices) with the attributes the bank reads."""

    def __init__(self, fs, idx):
        self.xy = np.asarray(fs.xy)[idx]
        self.descriptors = np.asarray(fs.descriptors)[idx]
        self.width, self.height = fs.width, fs.height

    def __len__(self):
        return len(self.xy)


def guided_match_pair(query_fs, target_fs, geom, *, d: float = BAND_D_PX,
                      ratio: float = RATIO_GUIDED, inflation: float = GRID_INFLATION,
                      strategy: str = "grid", query_indices=None, target_indices=None,
                      grid=None, single_cap: float = SINGLE_CANDIDATE_CAP,
                      stats: SearchStats | None = None) -> list:
    """Drop-in for msfm.guided.guided_match_pair (guided.py:393-480)."""
    ti = np.arange(len(target_fs)) if target_indices is None else np.asarray(target_indices)
    if len(ti) == 0:
        return []
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    D = float(grid.d) if grid is not None and hasattr(grid, "d") else d * inflation
    if D <= 0 and strategy == "grid":
        raise ValueError(f"cell half-size d must be positive, got {D}")
    if strategy != "grid":
        D = max(D, 1.0)   # the index is built but only grid mode consults its cells
    qi = np.arange(len(query_fs)) if query_indices is None else np.asarray(query_indices)
    qi = np.unique(qi.astype(np.int64))  # duplicates cannot change the match set
    if target_indices is None:
        tfs = target_fs
        bank = _pair_bank(query_fs, target_fs)
    else:
        tfs = _Sub(target_fs, ti)
        bank = FeatureBank({0: query_fs, 1: tfs})
    F = np.asarray(geom.F if hasattr(geom, "F") else geom, dtype=np.float64).reshape(1, 3, 3)
    with _DROPIN_LOCK:
        res = match_pairs(bank, [0], [1], F, [qi.astype(np.int32)], d=d, ratio=ratio,
                          grid_d=D, single_cap=single_cap, with_stats=stats is not None,
                          strategy=strategy)
        _, q, t, dist, rat = res.to_host()
        s = res.stats.cpu().numpy() if stats is not None else None
    if stats is not None:
        stats.add(int(s[0, 0]), int(s[0, 1]))
    qimg, timg = query_fs.image_id, target_fs.image_id
    return [Match(query=FeatureRef(qimg, int(a)), target=FeatureRef(timg, int(ti[b])),
                  distance=float(c), ratio=float(r))
            for a, b, c, r in zip(q, t, dist, rat)]
