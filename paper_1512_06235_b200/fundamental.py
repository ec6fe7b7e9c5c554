"""Robust two-view geometry on the device: estimate_fundamental_ransac
(geometry.py:153-198) batched over image pairs, plus the reference-shaped
drop-in.

Hypotheses are the reference's own numpy ``choice(n, 8)`` stream
(sampling.py / msfm_ransac_samples); the device fits and scores them all, the
adaptive stop (geometry.py:176-191, including its OverflowError) is replayed
on the host with the reference's numpy expressions, and the winner is refitted
on its inliers on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .pnp import _replay_batch
from .types import InsufficientDataError, TwoViewGeometry

SAMPSON_THRESHOLD_PX = 2.0     # geometry.py:19
RANSAC_CONFIDENCE = 0.999      # geometry.py:20
RANSAC_MAX_ITERS = 2048        # geometry.py:21
FIRST_ROUND = 256


@dataclass
class FResult:
    status: str                     # "ok" | "overflow" | "insufficient"
    F: np.ndarray | None = None
    mask: np.ndarray | None = None
    inlier_count: int = 0
    degenerate_planar: bool = False


class _Pairs:
    def __init__(self, dev, q_list, c_list):
        import torch

        self.n = np.array([len(x) for x in q_list], np.int64)
        off = np.zeros(len(q_list) + 1, np.int64)
        np.cumsum(self.n, out=off[1:])
        self.off_h = off
        q = np.concatenate([np.asarray(x, np.float64).reshape(-1, 2) for x in q_list])
        c = np.concatenate([np.asarray(x, np.float64).reshape(-1, 2) for x in c_list])

        def up(a):
            a = np.ascontiguousarray(a)
            return torch.from_numpy(a if a.size else np.zeros(1, a.dtype)).pin_memory().to(
                dev, non_blocking=True)

        self.q, self.c, self.off = up(q), up(c), up(off)


def _score(lib, pairs, samples, H, threshold, st, dev):
    import torch

    P = samples.shape[0]
    d_samples = torch.from_numpy(np.ascontiguousarray(samples)).pin_memory().to(dev, non_blocking=True)
    d_F = torch.empty((P, H, 9), dtype=torch.float64, device=dev)
    d_count = torch.empty((P, H), dtype=torch.int32, device=dev)
    _lib.check(lib.msfm_fundamental_hypotheses(_lib.ptr(pairs.q), _lib.ptr(pairs.c),
                                               _lib.ptr(pairs.off), P, _lib.ptr(d_samples), H,
                                               float(threshold), _lib.ptr(d_F), _lib.ptr(d_count),
                                               st), "msfm_fundamental_hypotheses")
    return d_F, d_count.cpu().numpy()


def fransac_batch(q_list, c_list, seeds, *, threshold=SAMPSON_THRESHOLD_PX,
                  confidence=RANSAC_CONFIDENCE, max_iters=RANSAC_MAX_ITERS, device=None,
                  stream=None, first_round=FIRST_ROUND):
    """estimate_fundamental_ransac for many pairs; one FResult per pair."""
    import torch

    lib = _lib.load()
    dev = torch.device(device or "cuda")
    B = len(q_list)
    results = [None] * B
    active = [i for i in range(B) if len(q_list[i]) >= 8]
    for i in range(B):
        if len(q_list[i]) < 8:
            results[i] = FResult("insufficient")
    if not active:
        return results
    pairs = _Pairs(dev, [q_list[i] for i in active], [c_list[i] for i in active])
    st = _lib.stream_handle(stream)
    A = len(active)
    H1 = min(max_iters, first_round)
    counts = np.full((A, max_iters), -2, np.int64)
    samples = np.zeros((A, H1, 8), np.int32)
    st_all = np.zeros((A, 6), np.uint64)
    if any(int(seeds[i]) < 0 for i in active):
        raise ValueError("expected non-negative integer seeds")   # as np.random.default_rng
    seed_arr = np.array([int(seeds[i]) for i in active], np.uint64)
    n_arr = np.ascontiguousarray(pairs.n, np.int64)
    _lib.check(lib.msfm_ransac_samples_seeded(A, seed_arr.ctypes.data, n_arr.ctypes.data, 8, H1,
                                              samples.ctypes.data, st_all.ctypes.data),
               "msfm_ransac_samples_seeded")
    states = [st_all[k] for k in range(A)]
    d_F1, c1 = _score(lib, pairs, samples, H1, threshold, st, dev)
    counts[:, :H1] = c1
    best = _replay_batch(counts, H1, pairs.n, max_iters, confidence, power=8)
    pending = [k for k in range(A) if best[k] != "overflow" and not best[k][4]]
    d_F2 = None
    if pending:
        H2 = max_iters - H1
        samples2 = np.zeros((len(pending), H2, 8), np.int32)
        for j, k in enumerate(pending):
            s6 = states[k]
            words = np.ascontiguousarray(s6[:4])
            _lib.check(lib.msfm_ransac_samples(words.ctypes.data, int(s6[4]), int(s6[5]),
                                               int(pairs.n[k]), 8, H2, samples2[j].ctypes.data,
                                               None), "msfm_ransac_samples")
        sub = _Pairs(dev, [q_list[active[k]] for k in pending], [c_list[active[k]] for k in pending])
        d_F2, c2 = _score(lib, sub, samples2, H2, threshold, st, dev)
        counts[pending, H1:] = c2
        for k, r in zip(pending, _replay_batch(counts[pending], max_iters, pairs.n[pending],
                                               max_iters, confidence, power=8)):
            best[k] = r
    status = np.zeros(A, np.int32)
    d_best = torch.zeros((A, 9), dtype=torch.float64, device=dev)
    src1, src2 = [], []
    for k in range(A):
        if best[k] == "overflow":
            results[active[k]] = FResult("overflow")
            continue
        bh, bc = best[k][0], best[k][1]
        if bh < 0 or bc < 8:
            # geometry.py:192-194: no usable hypothesis
            results[active[k]] = FResult("ok", np.eye(3) / np.sqrt(3.0),
                                         np.zeros(int(pairs.n[k]), bool), 0, False)
            continue
        status[k] = 1
        if bh < H1:
            src1.append((k, bh))
        else:
            src2.append((k, pending.index(k), bh - H1))
    if src1:
        ks = torch.tensor([x[0] for x in src1], device=dev)
        d_best[ks] = d_F1[ks, torch.tensor([x[1] for x in src1], device=dev)]
    if src2:
        ks = torch.tensor([x[0] for x in src2], device=dev)
        d_best[ks] = d_F2[torch.tensor([x[1] for x in src2], device=dev),
                          torch.tensor([x[2] for x in src2], device=dev)]
    if status.any():
        d_status = torch.from_numpy(status).to(dev)
        d_F = torch.zeros((A, 9), dtype=torch.float64, device=dev)
        d_mask = torch.zeros(max(int(pairs.off_h[-1]), 1), dtype=torch.uint8, device=dev)
        d_cnt = torch.zeros(A, dtype=torch.int32, device=dev)
        d_gap = torch.zeros(A, dtype=torch.float64, device=dev)
        _lib.check(lib.msfm_fundamental_refit(_lib.ptr(pairs.q), _lib.ptr(pairs.c),
                                              _lib.ptr(pairs.off), A, _lib.ptr(d_best),
                                              _lib.ptr(d_status), float(threshold), _lib.ptr(d_F),
                                              _lib.ptr(d_mask), _lib.ptr(d_cnt), _lib.ptr(d_gap),
                                              st), "msfm_fundamental_refit")
        F, mask, cnt, gap = (d_F.cpu().numpy(), d_mask.cpu().numpy(), d_cnt.cpu().numpy(),
                             d_gap.cpu().numpy())
        for k in range(A):
            if not status[k]:
                continue
            m = mask[pairs.off_h[k]:pairs.off_h[k + 1]].astype(bool)
            results[active[k]] = FResult("ok", F[k].reshape(3, 3).copy(), m, int(cnt[k]),
                                         bool(gap[k] < 1e-9))
    return results


def estimate_fundamental_ransac(pts_q, pts_c, *, threshold=SAMPSON_THRESHOLD_PX,
                                confidence=RANSAC_CONFIDENCE, max_iters=RANSAC_MAX_ITERS, seed=0):
    """Drop-in for msfm.geometry.estimate_fundamental_ransac: (TwoViewGeometry, mask);
    InsufficientDataError below 8 correspondences, OverflowError where the
    reference raises it (geometry.py:189)."""
    q = np.asarray(pts_q, dtype=np.float64).reshape(-1, 2)
    c = np.asarray(pts_c, dtype=np.float64).reshape(-1, 2)
    if len(q) < 8:
        raise InsufficientDataError(f"need >= 8 correspondences, got {len(q)}")
    r = fransac_batch([q], [c], [seed], threshold=threshold, confidence=confidence,
                      max_iters=max_iters)[0]
    if r.status == "overflow":
        raise OverflowError("cannot convert float infinity to integer")
    return TwoViewGeometry(F=r.F, inlier_count=r.inlier_count,
                           degenerate_planar=r.degenerate_planar), r.mask
