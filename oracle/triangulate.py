"""ORACLE — test infrastructure only (see oracle/__init__.py).

numpy restatement of msfm.geometry.triangulate_track (geometry.py:276-357):
DLT by SVD, one Gauss-Newton step, depth / error / angle gates."""

from __future__ import annotations

import numpy as np


class DegenerateGeometryError(Exception):
    pass


def triangulate(K, R, t, pix, max_error=4.0, min_angle_deg=1.0):
    """Returns ("ok", X, err) | ("rejected", None, None) | ("degenerate", None, None)."""
    n = len(K)
    centers = np.stack([-R[i].T @ t[i] for i in range(n)])
    if np.all(np.linalg.norm(centers - centers[0], axis=1) < 1e-12):
        return "degenerate", None, None
    P = [K[i] @ np.hstack([R[i], t[i].reshape(3, 1)]) for i in range(n)]
    A = np.zeros((2 * n, 4))
    for i in range(n):
        A[2 * i] = pix[i, 0] * P[i][2] - P[i][0]
        A[2 * i + 1] = pix[i, 1] * P[i][2] - P[i][1]
    Xh = np.linalg.svd(A)[2][-1]
    if abs(Xh[3]) < 1e-12 * np.linalg.norm(Xh[:3]):
        return "degenerate", None, None
    X = Xh[:3] / Xh[3]

    def reproject(Xw):
        res = np.zeros((n, 2))
        depths = np.zeros(n)
        for i in range(n):
            xc = R[i] @ Xw + t[i]
            depths[i] = xc[2]
            if xc[2] <= 1e-12:
                res[i] = np.inf
                continue
            uv = K[i] @ xc
            res[i] = uv[:2] / uv[2] - pix[i]
        return res, depths

    res, depths = reproject(X)
    err = float(np.mean(np.linalg.norm(res, axis=1))) if np.all(np.isfinite(res)) else np.inf
    if np.isfinite(err):
        J = np.zeros((2 * n, 3))
        for i in range(n):
            xc = R[i] @ X + t[i]
            f = K[i][0, 0]
            x, y, z = xc
            d_uv = np.array([[f / z, 0.0, -f * x / z ** 2], [0.0, f / z, -f * y / z ** 2]])
            J[2 * i:2 * i + 2] = d_uv @ R[i]
        r = res.reshape(-1)
        H = J.T @ J
        H[np.arange(3), np.arange(3)] += 1e-12
        try:
            X_new = X + np.linalg.solve(H, -(J.T @ r))
            res_new, depths_new = reproject(X_new)
            if np.all(np.isfinite(res_new)):
                err_new = float(np.mean(np.linalg.norm(res_new, axis=1)))
                if err_new <= err:
                    X, res, depths, err = X_new, res_new, depths_new, err_new
        except np.linalg.LinAlgError:
            pass
    if not np.isfinite(err) or np.any(depths <= 0) or err > max_error:
        return "rejected", None, None
    rays = X[None, :] - centers
    rays /= np.maximum(np.linalg.norm(rays, axis=1, keepdims=True), 1e-15)
    cosang = rays @ rays.T
    np.fill_diagonal(cosang, 1.0)
    if np.degrees(np.arccos(np.clip(cosang.min(), -1.0, 1.0))) < min_angle_deg:
        return "rejected", None, None
    return "ok", X, err
