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

    def packed_device(self, stream=None):
        """Like ``packed`` without the host sync: (rows int32 (cap, 4), total int64 (1,)
        on the device); rows past ``total`` are unspecified.  cap = the pair set's
        query count (one row per query at most)."""
        import torch

        lib = _lib.load()
        P = self.count.numel()
        dev = self.q.device
        off = torch.empty(P + 1, dtype=torch.int64, device=dev)
        rows = torch.empty((max(self.q.numel(), 1), 4), dtype=torch.int32, device=dev)
        if P:
            _lib.check(lib.msfm_pack_matches(P, _lib.ptr(self._qoff_d), _lib.ptr(self.count),
                                             _lib.ptr(self.q), _lib.ptr(self.t), _lib.ptr(self.dist),
                                             _lib.ptr(self.ratio), _lib.ptr(off), _lib.ptr(rows),
                                             _lib.stream_handle(stream)), "msfm_pack_matches")
        else:
            off.zero_()
        return rows, off[P:P + 1]

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
                     strategy: str = "grid", pinned=None, stage_plan=None,
                     first_chunk_pairs: int = 0):
    """``match_pairs`` + packing + one pinned host copy per internal chunk, the
    copy of chunk c overlapping the compute of chunk c+1 (msfm_guided_match_rows).
    Returns the host rows as a MATCH_ROW structured array (a view of ``pinned``
    when given: int32 (>= total queries, 4), pinned).  ``stage_plan``: the bank
    is still arriving (see match_pairs_rows_staged)."""
    import torch

    lib = _lib.load()
    if d <= 0:
        raise ValueError(f"cell half-size d must be positive, got {d}")
    if strategy not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}")
    D = float(grid_d) if grid_d is not None else float(d) * float(inflation)
    P = len(q_img)
    chunk_pairs = chunk_pairs or 1024       # several chunks: the readback overlaps compute
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
                           max(bank.max_n, 1), int(chunk_pairs), STRATEGIES[strategy],
                           int(first_chunk_pairs))
    qoff_c = np.ascontiguousarray(qoff, dtype=np.int64)
    ws_bytes = lib.msfm_guided_workspace_bytes(P, qoff_c.ctypes.data, ctypes.byref(prm))
    # scratch kept on the bank between calls of the same shape (a staged bank reused
    # step after step allocates nothing here after the first step)
    bufs = bank.__dict__.setdefault("_rows_bufs", {})

    def buf(name, shape, dtype, zero=False, pin=False):
        t = bufs.get(name)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = (torch.empty(shape, dtype=dtype, pin_memory=True) if pin
                 else torch.empty(shape, dtype=dtype, device=dev))
            bufs[name] = t
        if zero:
            t.zero_()
        return t

    ws = buf("ws", (max(ws_bytes, 1),), torch.uint8)
    cap = max(nq_total, 1)
    out_q = buf("q", (cap,), torch.int32)
    out_t = buf("t", (cap,), torch.int32)
    out_d = buf("d", (cap,), torch.float32)
    out_r = buf("r", (cap,), torch.float32)
    out_c = buf("c", (P,), torch.int32, zero=True)
    out_off = buf("off", (P + 1,), torch.int64)
    d_rows = buf("rows", (cap, 4), torch.int32)
    d_meta = buf("meta", (2 * (P + 1),), torch.int64, zero=True)
    h_meta = buf("hmeta", (2 * (P + 1),), torch.int64, zero=True, pin=True)
    if pinned is None or pinned.shape[0] < cap:
        pinned = torch.empty((cap, 4), dtype=torch.int32, pin_memory=True)
    total = ctypes.c_int64(0)
    copy_stream = bank.__dict__.get("_d2h_stream")
    if copy_stream is None:
        copy_stream = bank.__dict__["_d2h_stream"] = torch.cuda.Stream(device=dev)
    b, g = bank.cstruct(), grid.cstruct()
    _lib.check(lib.msfm_guided_match_rows(ctypes.byref(b), ctypes.byref(g), P, _lib.ptr(pq),
                                          _lib.ptr(pt), _lib.ptr(pF), _lib.ptr(qoff_d),
                                          _lib.ptr(qlist_d), _lib.ptr(qsrc_d), qoff_c.ctypes.data,
                                          ctypes.byref(prm), _lib.ptr(out_q), _lib.ptr(out_t),
                                          _lib.ptr(out_d), _lib.ptr(out_r), _lib.ptr(out_c),
                                          _lib.ptr(out_off), _lib.ptr(d_rows), _lib.ptr(d_meta),
                                          h_meta.data_ptr(), pinned.data_ptr(), ctypes.byref(total),
                                          _lib.ptr(ws), ws_bytes, _lib.stream_handle(stream),
                                          copy_stream.cuda_stream,
                                          ctypes.byref(stage_plan) if stage_plan else None),
               "msfm_guided_match_rows")
    n = int(total.value)
    return pinned[:n].numpy().view(MATCH_ROW).reshape(n)


def chunk_bounds(qoff, chunk_pairs: int = 0, max_nt: int = 1, first_chunk_pairs: int = 0):
    """The matcher's internal chunking (first pair of every chunk, then the end)."""
    lib = _lib.load(require_device=False)
    qoff_c = np.ascontiguousarray(qoff, dtype=np.int64)
    P = len(qoff_c) - 1
    prm = _lib.MatchParams(1.0, 1.0, 1.0, max(max_nt, 1), int(chunk_pairs), 0,
                           int(first_chunk_pairs))
    out = np.zeros(P + 2, np.int32)
    nc = lib.msfm_guided_chunk_bounds(P, qoff_c.ctypes.data, ctypes.byref(prm), out.ctypes.data,
                                      len(out))
    return out[:nc + 1].astype(np.int64)


def match_pairs_rows_staged(host, q_img, t_img, F, query_lists, *, device=None,
                            segment_images: int = 8, d: float = BAND_D_PX,
                            ratio: float = RATIO_GUIDED, inflation: float = GRID_INFLATION,
                            grid_d: float | None = None, single_cap: float = SINGLE_CANDIDATE_CAP,
                            chunk_pairs: int = 0, strategy: str = "grid", pinned=None,
                            first_chunk_pairs: int = 64, bank: FeatureBank | None = None,
                            host_pairs: HostPairs | None = None):
    """``match_pairs_rows`` straight from a pinned ``HostBank``, the upload
    pipelined into the matching: the bank goes up on a copy stream in ranges of
    ``segment_images`` images, in the order the matcher's chunks first read them;
    just before a chunk the matcher's stream waits for the ranges it first reads
    and indexes them (|desc|^2 + spatial index, msfm_stage_plan), so chunk c
    computes while later ranges are still in flight; a short first chunk
    (``first_chunk_pairs``) needs few ranges to start.  ``bank``: a staged bank
    from an earlier call over the same host bank, whose device buffers (rows,
    norms, spatial index) are refilled instead of allocated.  ``host_pairs``: the
    pair table already in pinned memory (``HostPairs``).  Returns (rows, bank)."""
    import torch

    lib = _lib.load()
    if d <= 0:
        raise ValueError(f"cell half-size d must be positive, got {d}")
    D = float(grid_d) if grid_d is not None else float(d) * float(inflation)
    P = len(q_img)
    # chunks of up to 1536 pairs (after the 64 / 256 / 1024 ramp): the upload and the
    # row readback pipeline across them (tools/probe_staged.py: 768 / 1024 / 1536 /
    # 2048-pair chunks 21.5 / 21.1 / 20.8 / 21.6 ms per C3 step)
    chunk_pairs = chunk_pairs or 1536
    if bank is None or not getattr(bank, "staged", False) or bank.host is not host:
        bank = FeatureBank(host=host, device=device, staged=True)
    nimg = len(bank.image_ids)
    seg = max(int(segment_images), 1)
    nseg = (nimg + seg - 1) // seg
    # H2D copies of all streams go through one copy engine in issue order: small
    # tables first, then the ranges the first chunk reads, then the pair tables
    # (prepared on the host while those land), then every other range
    grid = bank.grid(D, build=False)
    if host_pairs is not None:
        qoff = host_pairs.qoff
    else:
        lens = np.fromiter((len(x) for x in query_lists), dtype=np.int64, count=P)
        qoff = np.zeros(P + 1, dtype=np.int64)
        np.cumsum(lens, out=qoff[1:])
    # ranges in the order of the first chunk that reads them (host-only planning)
    bounds = (chunk_bounds(qoff, chunk_pairs, bank.max_n, first_chunk_pairs) if P
              else np.zeros(1, np.int64))
    nck = len(bounds) - 1
    qi, ti = bank.slots(q_img), bank.slots(t_img)
    first = np.full(nseg, max(nck - 1, 0), np.int64)      # unread ranges: before the last chunk
    for c in range(nck - 1, -1, -1):
        p0, p1 = int(bounds[c]), int(bounds[c + 1])
        first[np.unique(np.concatenate([qi[p0:p1], ti[p0:p1]]) // seg)] = c
    order = np.lexsort((np.arange(nseg), first))
    # neighbouring segments first read by the same chunk travel and index as one range
    k0l, k1l, chk = [], [], []
    for s in order:
        a, b = int(s) * seg, min((int(s) + 1) * seg, nimg)
        if k1l and k1l[-1] == a and chk[-1] == first[s]:
            k1l[-1] = b
        else:
            k0l.append(a)
            k1l.append(b)
            chk.append(int(first[s]))
    k0 = np.array(k0l, np.int32)
    k1 = np.array(k1l, np.int32)
    # one H2D stream per bank (torch's stream pool hands out a different stream per
    # call, each with its own allocator pool)
    copy_s = bank.__dict__.get("_h2d_stream")
    if copy_s is None:
        copy_s = bank.__dict__["_h2d_stream"] = torch.cuda.Stream(device=bank.device)
    copy_s.wait_stream(torch.cuda.current_stream(bank.device))
    if not bank.__dict__.get("_recorded"):
        bank.xy.record_stream(copy_s)
        bank.desc.record_stream(copy_s)
        bank.__dict__["_recorded"] = True
    n0 = int(np.searchsorted(np.array(chk), 1))           # ranges chunk 0 reads
    landed = [bank.upload_range(int(a), int(b), copy_s) for a, b in zip(k0[:n0], k1[:n0])]
    # the pair tables on the copy stream too, right behind chunk 0's ranges (the
    # matcher's stream waits for them: by then chunk 0's rows have landed as well)
    hp = host_pairs if host_pairs is not None else HostPairs(bank, q_img, t_img, F, query_lists)
    prev = bank.__dict__.get("_pairs_dev")
    reuse = prev[1] if prev is not None and prev[0] is hp else None
    inp = hp.upload(bank.device, copy_s, out=reuse)
    bank.__dict__["_pairs_dev"] = (hp, [inp[k] for k in (0, 1, 2, 3, 4, 6)])
    landed += [bank.upload_range(int(a), int(b), copy_s) for a, b in zip(k0[n0:], k1[n0:])]
    br = np.array([grid.bucket_range(int(a), int(b)) for a, b in zip(k0, k1)],
                  np.int64).reshape(-1, 2)
    fr = np.array([bank.row_range(int(a), int(b)) for a, b in zip(k0, k1)],
                  np.int64).reshape(-1, 2)
    arrs = dict(chunk=np.array(chk, np.int32), img0=k0, img1=k1,
                bucket0=np.ascontiguousarray(br[:, 0]), bucket1=np.ascontiguousarray(br[:, 1]),
                feat0=np.ascontiguousarray(fr[:, 0]), feat1=np.ascontiguousarray(fr[:, 1]))
    ev = (ctypes.c_void_p * max(len(landed), 1))(*[e._as_parameter_ for e in landed])
    plan = _lib.StagePlan(len(k0), *[arrs[k].ctypes.data for k in
                                         ("chunk", "img0", "img1", "bucket0", "bucket1",
                                          "feat0", "feat1")],
                          ctypes.cast(ev, ctypes.c_void_p), grid._nb, _lib.ptr(grid._ws),
                          grid._ws_bytes)
    plan._keep = (arrs, ev)
    if P == 0:
        # nothing to match: index the whole bank here so it is complete on return
        torch.cuda.current_stream(bank.device).wait_stream(copy_s)
        _lib.check(lib.msfm_feature_norms(_lib.ptr(bank.desc), bank.n_total, _lib.ptr(bank.norm2),
                                          _lib.stream_handle()), "msfm_feature_norms")
        grid.build_range(0, nimg)
        bank.pair_inputs = inp
        return np.zeros(0, MATCH_ROW), bank
    rows = match_pairs_rows(bank, q_img, t_img, F, query_lists, d=d, ratio=ratio,
                            inflation=inflation, grid_d=grid_d, single_cap=single_cap,
                            chunk_pairs=chunk_pairs, device_inputs=inp, strategy=strategy,
                            pinned=pinned, stage_plan=plan, first_chunk_pairs=first_chunk_pairs)
    bank.pair_inputs = inp
    bank._staging = copy_s
    return rows, bank


class HostPairs:
    """A matching step's pair table in pinned host memory (the H2D staging area
    next to ``HostBank``): bank slots of the query and target images, F, the
    query-list offsets, the query lists (a list object shared by several pairs —
    every pair of one query image, densify.py:150-158 — stored once) and each
    pair's list start.  ``upload`` is one copy per array."""

    def __init__(self, bank, q_img, t_img, F, query_lists):
        import torch

        P = len(q_img)
        self.n_pairs = P
        qi = bank.slots(q_img).astype(np.int32)
        ti = bank.slots(t_img).astype(np.int32)
        Fh = np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(P, 9))
        lens = np.fromiter((len(x) for x in query_lists), dtype=np.int64, count=P)
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
        self.qoff = qoff

        def pin(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()

        self.tensors = (pin(qi), pin(ti), pin(Fh), pin(qoff), pin(qlist), pin(src))

    @property
    def nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in self.tensors)

    def upload(self, dev, stream=None, out=None):
        """(q slots, t slots, F, qoff, qlist, qoff on the host, list starts) on ``dev``;
        with ``stream``: copied on that stream, and the current stream waits for them;
        ``out``: device tensors of an earlier upload of this table, refilled."""
        import torch

        if stream is None and out is None:
            qi, ti, Fh, qoff, qlist, src = (t.to(dev, non_blocking=True) for t in self.tensors)
            return (qi, ti, Fh, qoff, qlist, self.qoff, src)
        cur = torch.cuda.current_stream(dev)
        if out is None:
            # allocated in the current stream's pool (the one that consumes them)
            out = [torch.empty(tuple(t.shape), dtype=t.dtype, device=dev) for t in self.tensors]
        s = stream if stream is not None else cur
        with torch.cuda.stream(s):
            for d, h in zip(out, self.tensors):
                d.copy_(h, non_blocking=True)
        if s is not cur:
            cur.wait_stream(s)
        qi, ti, Fh, qoff, qlist, src = out
        return (qi, ti, Fh, qoff, qlist, self.qoff, src)


def prepare_pairs(bank: FeatureBank, q_img, t_img, F, query_lists):
    """Stage the pair table on the device (index translation + one copy per array).

    Query lists passed as the same object for several pairs (every pair of one
    query image, densify.py:150-158) are uploaded once and shared."""
    return HostPairs(bank, q_img, t_img, F, query_lists).upload(bank.device)

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
    # Python scalars first (.tolist()): f32 values widen exactly to float
    return [Match(query=FeatureRef(qimg, a), target=FeatureRef(timg, b), distance=c, ratio=r)
            for a, b, c, r in zip(np.asarray(q, np.int64).tolist(),
                                  np.asarray(ti)[np.asarray(t, np.int64)].astype(np.int64).tolist(),
                                  np.asarray(dist, np.float32).astype(np.float64).tolist(),
                                  np.asarray(rat, np.float32).astype(np.float64).tolist())]
