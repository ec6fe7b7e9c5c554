"""ORACLE — test infrastructure only (see oracle/__init__.py).

numpy restatements of the reference's 3D-2D localization path:

* ``knn2_exact`` — DescriptorIndex.knn2 exact path (descriptors.py:35-72) on the
  exact-integer form of the query means: a point with track-descriptor sum S
  and track length n (localize.py:51-59, mean = S/n) is ranked against image
  feature f by N = |S - n f|^2 = n^2 |S/n - f|^2 (int64, lowest index wins ties).
* ``direct_3d2d`` — direct_3d2d_search (localize.py:99-122) with ratio_filter
  (matching.py:82-103): accept iff sqrt(N_b)/sqrt(N_s) < ratio, evaluated
  exactly as q^2 N_b < p^2 N_s for ratio = p/q; single candidate: dist < cap;
  one point per feature by exact distance N/n^2 (lower point id wins ties).
* ``pnp_ransac`` / ``dlt_pose`` / ``refine_pose_lm`` — reconstruct.py:53-226,
  restated operation by operation (same numpy calls), including the
  OverflowError of reconstruct.py:210-211.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np


class InsufficientDataError(Exception):
    pass


def knn2_exact(S, n, F):
    """(idx_best, N_best, N_second) per point; N_second = -1 when F has 1 row."""
    if len(n) and int(np.max(n)) > 1000:
        # long tracks: N can pass 2^53, so every term in int64 (exact, slower)
        S = np.asarray(S, np.int64)
        n = np.asarray(n, np.int64)
        F = np.asarray(F, np.int64)
        N = ((S * S).sum(1)[:, None] - 2 * n[:, None] * (S @ F.T)
             + (n[:, None] ** 2) * (F * F).sum(1)[None, :])
    else:
        S = np.asarray(S, np.float64)
        n = np.asarray(n, np.float64)
        F = np.asarray(F, np.float64)
        SS = (S * S).sum(1)
        FF = (F * F).sum(1)
        # exact: every partial sum is an integer < 2^53
        N = SS[:, None] - 2.0 * n[:, None] * (S @ F.T) + (n[:, None] ** 2) * FF[None, :]
        N = np.rint(N).astype(np.int64)
    best = np.argmin(N, axis=1)
    rows = np.arange(len(N))
    nb = N[rows, best].copy()
    if N.shape[1] > 1:
        N[rows, best] = np.iinfo(np.int64).max
        ns = N.min(axis=1)
    else:
        ns = np.full(len(N), -1, np.int64)
    return best.astype(np.int64), nb, ns


def two_nearest(Q, T):
    """(dist f64 (n,2), idx i64 (n,2)) of descriptors.py:35-72 for integer-valued
    descriptors: integer squared distances (exact, as the reference's f32 BLAS
    form is for uint8 rows), argmin with the lowest index winning, the best
    column masked for the second, dist = sqrt in f32; +inf / -1 with one target."""
    Q = np.asarray(Q, np.int64).reshape(-1, 128)
    T = np.asarray(T, np.int64).reshape(-1, 128)
    nq, nt = len(Q), len(T)
    dist = np.full((nq, 2), np.inf)
    idx = np.full((nq, 2), -1, dtype=np.int64)
    if nq == 0 or nt == 0:
        return dist, idx
    d2 = (Q * Q).sum(1)[:, None] + (T * T).sum(1)[None, :] - 2 * (Q @ T.T)
    rows = np.arange(nq)
    best = np.argmin(d2, axis=1)
    dist[:, 0] = np.sqrt(d2[rows, best].astype(np.float32))
    idx[:, 0] = best
    if nt > 1:
        d2[rows, best] = np.iinfo(np.int64).max
        second = np.argmin(d2, axis=1)
        dist[:, 1] = np.sqrt(d2[rows, second].astype(np.float32))
        idx[:, 1] = second
    return dist, idx


def ratio_pq(ratio: float):
    f = Fraction(ratio).limit_denominator(1 << 20)
    return f.numerator, f.denominator


def direct_3d2d(point_ids, S, n, F, ratio=0.6, single_cap=45.0):
    """Sorted (pid, fid) correspondences."""
    point_ids = np.asarray(point_ids)
    if len(point_ids) == 0 or len(F) == 0:
        return np.zeros((0, 2), np.int64)
    idx, nb, ns = knn2_exact(S, n, F)
    p, q = ratio_pq(ratio)
    n64 = np.asarray(n, np.int64)
    acc = []
    for r in range(len(point_ids)):
        if ns[r] < 0:
            ok = np.sqrt(nb[r]) / n64[r] < single_cap
        else:
            ok = q * q * int(nb[r]) < p * p * int(ns[r])
        if ok:
            acc.append(r)
    best = {}
    for r in acc:
        f = int(idx[r])
        cur = best.get(f)
        # exact distance compare N1/n1^2 < N2/n2^2 (strict: the lower pid keeps ties)
        if cur is None or int(nb[r]) * int(n64[cur]) ** 2 < int(nb[cur]) * int(n64[r]) ** 2:
            best[f] = r
    out = sorted((int(point_ids[r]), f) for f, r in best.items())
    return np.array(out, np.int64).reshape(-1, 2)


# ------------------------------------------------------------------ PnP ---

def rodrigues(w):
    theta = np.linalg.norm(w)
    if theta < 1e-12:
        W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], dtype=np.float64)
        return np.eye(3) + W
    k = w / theta
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(theta) * K + (1.0 - np.cos(theta)) * (K @ K)


def dlt_pose(points3d, pixels, K):
    X = np.asarray(points3d, dtype=np.float64)
    uv = np.asarray(pixels, dtype=np.float64)
    n = len(X)
    if n < 6:
        raise InsufficientDataError(f"resection needs >= 6 points, got {n}")
    cx = X.mean(axis=0)
    sx = np.sqrt(3.0) / max(np.linalg.norm(X - cx, axis=1).mean(), 1e-12)
    cu = uv.mean(axis=0)
    su = np.sqrt(2.0) / max(np.linalg.norm(uv - cu, axis=1).mean(), 1e-12)
    Xn = (X - cx) * sx
    un = (uv - cu) * su
    A = np.zeros((2 * n, 12))
    Xh = np.hstack([Xn, np.ones((n, 1))])
    A[0::2, 0:4] = Xh
    A[0::2, 8:12] = -un[:, 0:1] * Xh
    A[1::2, 4:8] = Xh
    A[1::2, 8:12] = -un[:, 1:2] * Xh
    _, _, Vt = np.linalg.svd(A)
    Pn = Vt[-1].reshape(3, 4)
    Tu = np.array([[su, 0, -su * cu[0]], [0, su, -su * cu[1]], [0, 0, 1.0]])
    Tx = np.eye(4)
    Tx[:3, :3] *= sx
    Tx[:3, 3] = -sx * cx
    P = np.linalg.inv(Tu) @ Pn @ Tx
    G = np.linalg.inv(K) @ P
    best = None
    for sign in (1.0, -1.0):
        M = sign * G[:, :3]
        U, Sv, Vt2 = np.linalg.svd(M)
        R = U @ Vt2
        if np.linalg.det(R) < 0:
            continue
        scale = Sv.mean()
        if scale < 1e-12:
            continue
        t = sign * G[:, 3] / scale
        depths = (X @ R.T + t)[:, 2]
        front = int((depths > 0).sum())
        if best is None or front > best[0]:
            best = (front, R, t)
    if best is None or best[0] == 0:
        raise InsufficientDataError("resection produced no valid orientation")
    return best[1], best[2]


def refine_pose_lm(R, t, K, points3d, pixels, iters=20):
    X = np.asarray(points3d, dtype=np.float64)
    uv = np.asarray(pixels, dtype=np.float64)
    f = K[0, 0]
    pp = K[:2, 2]

    def residuals(Rc, tc):
        xc = X @ Rc.T + tc
        return f * xc[:, :2] / xc[:, 2:3] + pp - uv, xc

    res, xc = residuals(R, t)
    cost = float((res ** 2).sum())
    lam = 1e-6
    for _ in range(iters):
        x, y, z = xc[:, 0], xc[:, 1], xc[:, 2]
        d_uv = np.zeros((len(X), 2, 3))
        d_uv[:, 0, 0] = f / z
        d_uv[:, 0, 2] = -f * x / z ** 2
        d_uv[:, 1, 1] = f / z
        d_uv[:, 1, 2] = -f * y / z ** 2
        RX = xc - t
        d_rot = np.zeros((len(X), 3, 3))
        d_rot[:, 0, 1] = RX[:, 2]
        d_rot[:, 0, 2] = -RX[:, 1]
        d_rot[:, 1, 0] = -RX[:, 2]
        d_rot[:, 1, 2] = RX[:, 0]
        d_rot[:, 2, 0] = RX[:, 1]
        d_rot[:, 2, 1] = -RX[:, 0]
        J = np.zeros((len(X), 2, 6))
        J[:, :, 0:3] = d_uv @ d_rot
        J[:, :, 3:6] = d_uv
        Jf = J.reshape(-1, 6)
        rf = res.reshape(-1)
        H = Jf.T @ Jf
        g = Jf.T @ rf
        stepped = False
        for _ in range(8):
            Hd = H + lam * np.diag(np.maximum(np.diag(H), 1e-12))
            try:
                delta = np.linalg.solve(Hd, -g)
            except np.linalg.LinAlgError:
                lam *= 10.0
                continue
            R_new = rodrigues(delta[0:3]) @ R
            t_new = t + delta[3:6]
            res_new, xc_new = residuals(R_new, t_new)
            cost_new = float((res_new ** 2).sum())
            if np.isfinite(cost_new) and cost_new < cost:
                rel = (cost - cost_new) / max(cost, 1e-30)
                R, t, res, xc, cost = R_new, t_new, res_new, xc_new, cost_new
                lam = max(lam / 10.0, 1e-15)
                stepped = True
                if rel < 1e-10:
                    return R, t
                break
            lam *= 10.0
        if not stepped:
            break
    return R, t


def pnp_ransac(points3d, pixels, K, *, threshold=4.0, min_inliers=16, max_iters=2048,
               confidence=0.999, seed=0):
    X = np.asarray(points3d, dtype=np.float64).reshape(-1, 3)
    uv = np.asarray(pixels, dtype=np.float64).reshape(-1, 2)
    n = len(X)
    if n < 6:
        raise InsufficientDataError(f"resection needs >= 6 correspondences, got {n}")
    rng = np.random.default_rng(seed)
    f = K[0, 0]
    pp = K[:2, 2]
    best_mask = None
    best_count = 0
    needed = max_iters
    it = 0
    while it < needed and it < max_iters:
        it += 1
        sample = rng.choice(n, size=6, replace=False)
        try:
            R, t = dlt_pose(X[sample], uv[sample], K)
        except (InsufficientDataError, np.linalg.LinAlgError):
            continue
        xc = X @ R.T + t
        with np.errstate(divide="ignore", invalid="ignore"):
            proj = f * xc[:, :2] / xc[:, 2:3] + pp
            err = np.linalg.norm(proj - uv, axis=1)
        mask = (xc[:, 2] > 0) & np.isfinite(err) & (err < threshold)
        count = int(mask.sum())
        if count > best_count:
            best_count = count
            best_mask = mask
            w = count / n
            if w > 0:
                with np.errstate(divide="ignore"):
                    denom = np.log(max(1.0 - w ** 6, 1e-15))
                    needed = min(max_iters, int(np.ceil(np.log(1.0 - confidence) / denom)))
    if best_mask is None or best_count < max(min_inliers, 6):
        return None
    try:
        R, t = dlt_pose(X[best_mask], uv[best_mask], K)
    except (InsufficientDataError, np.linalg.LinAlgError):
        return None
    R, t = refine_pose_lm(R, t, K, X[best_mask], uv[best_mask])
    xc = X @ R.T + t
    with np.errstate(divide="ignore", invalid="ignore"):
        proj = f * xc[:, :2] / xc[:, 2:3] + pp
        err = np.linalg.norm(proj - uv, axis=1)
    mask = (xc[:, 2] > 0) & np.isfinite(err) & (err < threshold)
    if int(mask.sum()) < min_inliers:
        return None
    return R, t, mask
