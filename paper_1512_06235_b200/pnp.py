"""PnP-RANSAC on the device, batched over images, plus the reference-shaped
``pnp_ransac`` drop-in (reconstruct.py:168-226).

Hypotheses are the reference's own numpy ``choice`` stream (sampling.py); the
device scores them all, the adaptive stop (``needed``, reconstruct.py:192-211,
including its OverflowError) is replayed here with the reference's exact
numpy expressions, and the winning pose is refitted + LM-refined on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .types import InsufficientDataError

PNP_THRESHOLD_PX = 4.0
PNP_MIN_INLIERS = 16
PNP_MAX_ITERS = 2048
PNP_CONFIDENCE = 0.999
FIRST_ROUND = 256


@dataclass
class PnpResult:
    status: str            # "ok" | "none" | "overflow" | "insufficient"
    R: np.ndarray | None = None
    t: np.ndarray | None = None
    mask: np.ndarray | None = None
    iterations: int = 0


def _replay(counts, evaluated, n, max_iters, confidence, power=6):
    """The reference's while-loop over hypothesis outcomes (reconstruct.py:190-211;
    geometry.py:176-191 with power 8).  Returns (best_h, best_count, it, needed,
    complete); stops early when it runs past the evaluated hypotheses."""
    best_count, best_h, needed, it = 0, -1, max_iters, 0
    while it < needed and it < max_iters:
        if it >= evaluated:
            return best_h, best_count, it, needed, False
        h = it
        it += 1
        c = int(counts[h])
        if c < 0:
            continue
        if c > best_count:
            best_count, best_h = c, h
            w = c / n
            if w > 0:
                with np.errstate(divide="ignore"):
                    denom = np.log(max(1.0 - w ** power, 1e-15))
                    needed = min(max_iters, int(np.ceil(np.log(1.0 - confidence) / denom)))
    return best_h, best_count, it, needed, True


def _replay_records(counts, evaluated, n, max_iters, confidence, power=6):
    """_replay visiting only the improving hypotheses ("records"): the loop state
    changes nowhere else, so the same scalar numpy expressions are evaluated in
    the same order and the result (including the OverflowError) is identical."""
    c = np.asarray(counts[:evaluated], np.int64)
    prev = np.maximum.accumulate(np.concatenate([[0], np.maximum(c, 0)]))[:-1]
    recs = np.flatnonzero(c > prev)
    best_count, best_h, needed = 0, -1, max_iters
    for h in recs.tolist():
        if h >= needed or h >= max_iters:
            break                                   # the loop stopped before h
        cnt = int(c[h])
        best_count, best_h = cnt, h
        w = cnt / n
        if w > 0:
            with np.errstate(divide="ignore"):
                denom = np.log(max(1.0 - w ** power, 1e-15))
                needed = min(max_iters, int(np.ceil(np.log(1.0 - confidence) / denom)))
    stop = min(needed, max_iters)
    last = best_h + 1
    it = max(stop, last) if best_h >= 0 and last > stop else stop
    if it > evaluated:
        return best_h, best_count, evaluated, needed, False
    return best_h, best_count, it, needed, True


def _replay_batch(counts, evaluated, n, max_iters, confidence, power=6):
    """_replay_records for every row of ``counts`` (A, >= evaluated).  The record
    positions of all rows come from one vectorized pass; the reference's
    ``needed`` at every record is evaluated once for all rows: ``1 - w**power``
    and the max with 1e-15 as the Python float expressions, then np.log / divide
    / ceil on one array (numpy's float64 ufunc loop is the one its scalar calls
    run, so the values are the reference's bit for bit; a non-finite quotient is
    the reference's OverflowError).  Per row only the integer scan remains.
    Returns, per row, the _replay tuple or "overflow"."""
    C = np.asarray(counts)[:, :evaluated].astype(np.int64)
    A = C.shape[0]
    prev = np.maximum.accumulate(np.concatenate([np.zeros((A, 1), np.int64), np.maximum(C, 0)],
                                                axis=1), axis=1)[:, :-1]
    rr, cc = np.nonzero(C > prev)
    starts = np.searchsorted(rr, np.arange(A + 1)).tolist()
    cc_l, cnt_l = cc.tolist(), C[rr, cc].tolist()
    n_l = np.asarray(n, np.int64)[rr].tolist()
    # records have count >= 1, so w > 0 and the reference always evaluates needed
    arg = np.array([max(1.0 - (c / m) ** power, 1e-15) for c, m in zip(cnt_l, n_l)], np.float64)
    with np.errstate(divide="ignore"):
        quo = np.ceil(np.log(1.0 - confidence) / np.log(arg))
    ovf_l = (~np.isfinite(quo)).tolist()
    need_l = np.where(np.isfinite(quo), np.minimum(np.nan_to_num(quo, posinf=0.0, neginf=0.0),
                                                   max_iters), 0).astype(np.int64).tolist()
    out = []
    for k in range(A):
        best_count, best_h, needed, ovf = 0, -1, max_iters, False
        for j in range(starts[k], starts[k + 1]):
            h = cc_l[j]
            if h >= needed or h >= max_iters:
                break
            best_count, best_h = cnt_l[j], h
            if ovf_l[j]:
                ovf = True
                break
            needed = need_l[j]
        if ovf:
            out.append("overflow")
            continue
        stop = min(needed, max_iters)
        last = best_h + 1
        it = max(stop, last) if best_h >= 0 and last > stop else stop
        if it > evaluated:
            out.append((best_h, best_count, evaluated, needed, False))
        else:
            out.append((best_h, best_count, it, needed, True))
    return out


class _Batch:
    def __init__(self, dev, X_list, uv_list, K_list, flat=None):
        """Correspondences of many images as one device batch: per-image lists, or
        ``flat`` = (X (N,3), uv (N,2), offsets (B+1,)) already concatenated."""
        import torch

        if flat is not None:
            X, uv, off = flat
            off = np.asarray(off, np.int64)
            self.n = np.diff(off)
        else:
            self.n = np.array([len(x) for x in X_list], dtype=np.int64)
            off = np.zeros(len(X_list) + 1, np.int64)
            np.cumsum(self.n, out=off[1:])
            X = np.concatenate([np.asarray(x, np.float64).reshape(-1, 3) for x in X_list]) \
                if len(X_list) else np.zeros((0, 3))
            uv = np.concatenate([np.asarray(u, np.float64).reshape(-1, 2) for u in uv_list]) \
                if len(uv_list) else np.zeros((0, 2))
        self.off_h = off
        K = np.stack([np.asarray(k, np.float64).reshape(9) for k in K_list]) \
            if len(K_list) else np.zeros((0, 9))

        def up(a, cols):
            if isinstance(a, torch.Tensor):          # already on the device (e.g. gathered there)
                a = a.to(device=dev, dtype=torch.float64).reshape(-1, cols).contiguous()
                return a if a.numel() else torch.zeros((1, cols), dtype=torch.float64, device=dev)
            a = np.ascontiguousarray(a, np.float64).reshape(-1, cols)
            if a.size == 0:
                a = np.zeros((1, cols), a.dtype)
            return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)

        def up_i(a):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, a.dtype)
            return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)

        self.X, self.uv = up(X, 3), up(uv, 2)
        self.off, self.K = up_i(off), up_i(K)

    def subset(self, dev, rows, K_list):
        import torch

        sel = np.concatenate([np.arange(self.off_h[k], self.off_h[k + 1]) for k in rows]) \
            if len(rows) else np.zeros(0, np.int64)
        off = np.zeros(len(rows) + 1, np.int64)
        np.cumsum(self.n[rows], out=off[1:])
        d_sel = _lib.h2d(sel, dev)
        return _Batch(dev, None, None, K_list, flat=(self.X[d_sel], self.uv[d_sel], off))


def pnp_batch_flat(X, uv, off, K_list, seeds, **kw):
    """pnp_batch over concatenated correspondences: image k owns rows
    [off[k], off[k+1]) of X (N,3) and uv (N,2)."""
    return pnp_batch(None, None, K_list, seeds, flat=(X, uv, off), **kw)


def pnp_batch(X_list, uv_list, K_list, seeds, *, threshold=PNP_THRESHOLD_PX,
              min_inliers=PNP_MIN_INLIERS, max_iters=PNP_MAX_ITERS,
              confidence=PNP_CONFIDENCE, device=None, stream=None, first_round=FIRST_ROUND,
              flat=None, timing=None):
    """pnp_ransac for many images; returns a PnpResult per image.  Images with
    fewer than 6 correspondences get status "insufficient" (the reference raises
    InsufficientDataError there)."""
    import torch

    lib = _lib.load()
    dev = torch.device(device or "cuda")

    def mark(name):
        # optional phase timing (tools/probe_localize.py): device synchronized
        if timing is not None:
            import time
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            timing[name] = timing.get(name, 0.0) + (t - timing.get("_t", t))
            timing["_t"] = t

    mark("_start")
    if flat is not None:
        sizes = np.diff(np.asarray(flat[2], np.int64))
    else:
        sizes = np.array([len(x) for x in X_list], np.int64)
    B = len(sizes)
    results = [None] * B
    active = [i for i in range(B) if sizes[i] >= 6]
    for i in range(B):
        if sizes[i] < 6:
            results[i] = PnpResult("insufficient")
    if not active:
        return results
    if flat is not None:
        full = _Batch(dev, None, None, K_list, flat=flat) if len(active) == B else None
        batch = full if full is not None else \
            _Batch(dev, None, None, [], flat=flat).subset(dev, active, [K_list[i] for i in active])
    else:
        batch = _Batch(dev, [X_list[i] for i in active], [uv_list[i] for i in active],
                       [K_list[i] for i in active])
    st = _lib.stream_handle(stream)
    A = len(active)
    H1 = min(max_iters, first_round)
    mark("batch upload")
    counts = np.full((A, max_iters), -2, np.int64)
    # every stream's default_rng(seed).choice draws generated on the device (one
    # thread per stream; the PCG64 / SeedSequence restatement shared with the host
    # sampler), straight into the hypothesis kernel's input
    if any(int(seeds[i]) < 0 for i in active):
        raise ValueError("expected non-negative integer seeds")   # as np.random.default_rng
    seed_arr = np.array([int(seeds[i]) for i in active], np.uint64)
    n_arr = np.ascontiguousarray(batch.n, np.int64)
    d_samples = torch.empty((A, H1, 6), dtype=torch.int32, device=dev)
    d_state = torch.empty((A, 6), dtype=torch.int64, device=dev)
    d_bad = torch.zeros(1 + A, dtype=torch.int32, device=dev)
    # named: a temporary's block could be handed to the next allocation before the
    # kernel reads it
    d_seeds, d_n = _lib.h2d(seed_arr.view(np.int64), dev), _lib.h2d(n_arr, dev)
    _lib.check(lib.msfm_ransac_samples_seeded_device(
        A, _lib.ptr(d_seeds), _lib.ptr(d_n), 6, H1,
        _lib.ptr(d_samples), _lib.ptr(d_state), _lib.ptr(d_bad), st),
        "msfm_ransac_samples_seeded_device")
    mark("samples (device)")
    # hypotheses stay on the device; only the inlier counts come back for the replay
    d_hyp1, c1 = _score(lib, batch, d_samples, H1, threshold, st, dev)
    if int(d_bad[0].item()):
        raise ValueError("RANSAC population outside numpy choice's Floyd branch")
    counts[:, :H1] = c1
    mark("round 1 score")
    best = _replay_batch(counts, H1, batch.n, max_iters, confidence)
    mark("round 1 replay")
    pending = [k for k in range(A) if best[k] != "overflow" and not best[k][4]]
    d_hyp2 = None
    if pending:
        st_all = d_state.cpu().numpy().view(np.uint64)
        states = [(st_all[k],) for k in range(A)]
        # second round: continue each stream up to the current `needed` bound
        H2 = max_iters - H1
        samples2 = np.zeros((len(pending), H2, 6), np.int32)
        for j, k in enumerate(pending):
            st6 = states[k][0]
            words = np.ascontiguousarray(st6[:4])
            _lib.check(lib.msfm_ransac_samples(words.ctypes.data, int(st6[4]), int(st6[5]),
                                               int(batch.n[k]), 6, H2, samples2[j].ctypes.data,
                                               None), "msfm_ransac_samples")
        sub = batch.subset(dev, pending, [K_list[active[k]] for k in pending])
        d_hyp2, c2 = _score(lib, sub, samples2, H2, threshold, st, dev)
        counts[pending, H1:] = c2
        for k, r in zip(pending, _replay_batch(counts[pending], max_iters, batch.n[pending],
                                               max_iters, confidence)):
            best[k] = r
        mark(f"round 2 ({len(pending)} images)")
    # refit the winners: gather each winning hypothesis on the device
    import torch

    status = np.zeros(A, np.int32)
    src1, src2 = [], []
    for k in range(A):
        if best[k] == "overflow":
            results[active[k]] = PnpResult("overflow")
            continue
        bh, bc, it, _, _ = best[k]
        if bh < 0 or bc < max(min_inliers, 6):
            results[active[k]] = PnpResult("none", iterations=it)
            continue
        status[k] = 1
        if bh < H1:
            src1.append((k, bh))
        else:
            src2.append((k, pending.index(k), bh - H1))
    if status.any():
        d_best = torch.zeros((A, 12), dtype=torch.float64, device=dev)
        if src1:
            s1 = np.array(src1, np.int64).reshape(-1, 2)
            ks = _lib.h2d(s1[:, 0], dev)
            d_best[ks] = d_hyp1.reshape(-1, 12)[_lib.h2d(s1[:, 0] * H1 + s1[:, 1], dev)]
        if src2:
            s2 = np.array(src2, np.int64).reshape(-1, 3)
            ks = _lib.h2d(s2[:, 0], dev)
            d_best[ks] = d_hyp2.reshape(-1, 12)[_lib.h2d(s2[:, 1] * d_hyp2.shape[1] + s2[:, 2], dev)]
        _refit(lib, batch, status, d_best, threshold, min_inliers, st, dev, results, active, best)
    mark("refit + results")
    return results


def _score(lib, batch, samples, H, threshold, st, dev):
    """Device hypotheses (A, H, 12) and host inlier counts (A, H)."""
    import torch

    A = samples.shape[0]
    if not isinstance(samples, torch.Tensor):
        samples = torch.from_numpy(np.ascontiguousarray(samples)).pin_memory()
    d_samples = samples.to(dev, non_blocking=True)
    d_hyp = torch.empty((A, H, 12), dtype=torch.float64, device=dev)
    d_count = torch.empty((A, H), dtype=torch.int32, device=dev)
    _lib.check(lib.msfm_pnp_hypotheses(_lib.ptr(batch.X), _lib.ptr(batch.uv), _lib.ptr(batch.off),
                                       _lib.ptr(batch.K), A, _lib.ptr(d_samples), H,
                                       float(threshold), _lib.ptr(d_hyp), _lib.ptr(d_count), st),
               "msfm_pnp_hypotheses")
    return d_hyp, d_count.cpu().numpy()


def _refit(lib, batch, status, d_best, threshold, min_inliers, st, dev, results, active, best):
    import torch

    A = len(status)
    d_status = _lib.h2d(status, dev)
    d_R = torch.zeros((A, 9), dtype=torch.float64, device=dev)
    d_t = torch.zeros((A, 3), dtype=torch.float64, device=dev)
    d_mask = torch.zeros(max(int(batch.off_h[-1]), 1), dtype=torch.uint8, device=dev)
    d_ni = torch.zeros(A, dtype=torch.int32, device=dev)
    d_ok = torch.zeros(A, dtype=torch.int32, device=dev)
    _lib.check(lib.msfm_pnp_refit(_lib.ptr(batch.X), _lib.ptr(batch.uv), _lib.ptr(batch.off),
                                  _lib.ptr(batch.K), A, _lib.ptr(d_best), _lib.ptr(d_status),
                                  float(threshold), int(min_inliers), 20, _lib.ptr(d_R),
                                  _lib.ptr(d_t), _lib.ptr(d_mask), _lib.ptr(d_ni), _lib.ptr(d_ok), st),
               "msfm_pnp_refit")
    # two copies back: (R | t | ok) rows and the inlier masks
    pose = torch.cat([d_R, d_t, d_ok.to(torch.float64)[:, None]], dim=1).cpu().numpy()
    mask = d_mask.cpu().numpy()
    R, t, ok = pose[:, :9], pose[:, 9:12], pose[:, 12] != 0
    for k in range(A):
        if not status[k]:
            continue
        it = best[k][2]
        if ok[k]:
            m = mask[batch.off_h[k]:batch.off_h[k + 1]].astype(bool)
            results[active[k]] = PnpResult("ok", R[k].reshape(3, 3).copy(), t[k].copy(), m, it)
        else:
            results[active[k]] = PnpResult("none", iterations=it)


def pnp_ransac(points3d, pixels, K, *, threshold=PNP_THRESHOLD_PX, min_inliers=PNP_MIN_INLIERS,
               max_iters=PNP_MAX_ITERS, confidence=PNP_CONFIDENCE, seed=0):
    """Drop-in for msfm.reconstruct.pnp_ransac: (R, t, inlier_mask) or None;
    InsufficientDataError below 6 correspondences; OverflowError where the
    reference raises it (reconstruct.py:210-211)."""
    X = np.asarray(points3d, dtype=np.float64).reshape(-1, 3)
    uv = np.asarray(pixels, dtype=np.float64).reshape(-1, 2)
    if len(X) < 6:
        raise InsufficientDataError(f"resection needs >= 6 correspondences, got {len(X)}")
    r = pnp_batch([X], [uv], [np.asarray(K, np.float64)], [seed], threshold=threshold,
                  min_inliers=min_inliers, max_iters=max_iters, confidence=confidence)[0]
    if r.status == "overflow":
        raise OverflowError("cannot convert float infinity to integer")
    if r.status != "ok":
        return None
    return r.R, r.t, r.mask
