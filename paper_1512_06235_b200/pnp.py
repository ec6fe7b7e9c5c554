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


class _Batch:
    def __init__(self, dev, X_list, uv_list, K_list):
        import torch

        self.n = np.array([len(x) for x in X_list], dtype=np.int64)
        off = np.zeros(len(X_list) + 1, np.int64)
        np.cumsum(self.n, out=off[1:])
        self.off_h = off
        X = np.concatenate([np.asarray(x, np.float64).reshape(-1, 3) for x in X_list]) \
            if len(X_list) else np.zeros((0, 3))
        uv = np.concatenate([np.asarray(u, np.float64).reshape(-1, 2) for u in uv_list]) \
            if len(uv_list) else np.zeros((0, 2))
        K = np.stack([np.asarray(k, np.float64).reshape(9) for k in K_list]) \
            if len(K_list) else np.zeros((0, 9))

        def up(a):
            a = np.ascontiguousarray(a)
            if a.size == 0:
                a = np.zeros(1, a.dtype)
            return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)

        self.X, self.uv, self.off, self.K = up(X), up(uv), up(off), up(K)


def pnp_batch(X_list, uv_list, K_list, seeds, *, threshold=PNP_THRESHOLD_PX,
              min_inliers=PNP_MIN_INLIERS, max_iters=PNP_MAX_ITERS,
              confidence=PNP_CONFIDENCE, device=None, stream=None, first_round=FIRST_ROUND):
    """pnp_ransac for many images; returns a PnpResult per image.  Images with
    fewer than 6 correspondences get status "insufficient" (the reference raises
    InsufficientDataError there)."""
    import torch

    lib = _lib.load()
    dev = torch.device(device or "cuda")
    B = len(X_list)
    results = [None] * B
    active = [i for i in range(B) if len(X_list[i]) >= 6]
    for i in range(B):
        if len(X_list[i]) < 6:
            results[i] = PnpResult("insufficient")
    if not active:
        return results
    batch = _Batch(dev, [X_list[i] for i in active], [uv_list[i] for i in active],
                   [K_list[i] for i in active])
    st = _lib.stream_handle(stream)
    A = len(active)
    H1 = min(max_iters, first_round)
    counts = np.full((A, max_iters), -2, np.int64)
    # all streams default_rng(seed) at once (SeedSequence restated natively)
    samples = np.zeros((A, H1, 6), np.int32)
    st_all = np.zeros((A, 6), np.uint64)
    if any(int(seeds[i]) < 0 for i in active):
        raise ValueError("expected non-negative integer seeds")   # as np.random.default_rng
    seed_arr = np.array([int(seeds[i]) for i in active], np.uint64)
    n_arr = np.ascontiguousarray(batch.n, np.int64)
    _lib.check(lib.msfm_ransac_samples_seeded(A, seed_arr.ctypes.data, n_arr.ctypes.data, 6, H1,
                                              samples.ctypes.data, st_all.ctypes.data),
               "msfm_ransac_samples_seeded")
    states = [(st_all[k],) for k in range(A)]
    # hypotheses stay on the device; only the inlier counts come back for the replay
    d_hyp1, c1 = _score(lib, batch, samples, H1, threshold, st, dev)
    counts[:, :H1] = c1
    best = [None] * A
    pending = []
    for k in range(A):
        try:
            r = _replay(counts[k], H1, int(batch.n[k]), max_iters, confidence)
        except OverflowError:
            best[k] = "overflow"
            continue
        if r[4]:
            best[k] = r
        else:
            pending.append(k)
    d_hyp2 = None
    if pending:
        # second round: continue each stream up to the current `needed` bound
        H2 = max_iters - H1
        samples2 = np.zeros((len(pending), H2, 6), np.int32)
        for j, k in enumerate(pending):
            st6 = states[k][0]
            words = np.ascontiguousarray(st6[:4])
            _lib.check(lib.msfm_ransac_samples(words.ctypes.data, int(st6[4]), int(st6[5]),
                                               int(batch.n[k]), 6, H2, samples2[j].ctypes.data,
                                               None), "msfm_ransac_samples")
        sub = _Batch(dev, [np.asarray(X_list[active[k]]) for k in pending],
                     [np.asarray(uv_list[active[k]]) for k in pending],
                     [K_list[active[k]] for k in pending])
        d_hyp2, c2 = _score(lib, sub, samples2, H2, threshold, st, dev)
        for j, k in enumerate(pending):
            counts[k, H1:] = c2[j]
            try:
                r = _replay(counts[k], max_iters, int(batch.n[k]), max_iters, confidence)
            except OverflowError:
                best[k] = "overflow"
                continue
            best[k] = r
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
            ks = torch.tensor([x[0] for x in src1], device=dev)
            hs = torch.tensor([x[1] for x in src1], device=dev)
            d_best[ks] = d_hyp1[ks, hs]
        if src2:
            ks = torch.tensor([x[0] for x in src2], device=dev)
            js = torch.tensor([x[1] for x in src2], device=dev)
            hs = torch.tensor([x[2] for x in src2], device=dev)
            d_best[ks] = d_hyp2[js, hs]
        _refit(lib, batch, status, d_best, threshold, min_inliers, st, dev, results, active, best)
    return results


def _score(lib, batch, samples, H, threshold, st, dev):
    """Device hypotheses (A, H, 12) and host inlier counts (A, H)."""
    import torch

    A = samples.shape[0]
    d_samples = torch.from_numpy(np.ascontiguousarray(samples)).pin_memory().to(dev, non_blocking=True)
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
    d_status = torch.from_numpy(status).to(dev)
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
    R, t, mask, ok = d_R.cpu().numpy(), d_t.cpu().numpy(), d_mask.cpu().numpy(), d_ok.cpu().numpy()
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
