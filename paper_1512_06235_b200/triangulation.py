"""Multi-view DLT triangulation on the device (geometry.py:276-357), batched
over tracks, plus the reference-shaped ``triangulate_track`` drop-in."""

from __future__ import annotations

import numpy as np

from . import _lib
from .types import DegenerateGeometryError, InsufficientDataError, Triangulated

TRI_MAX_ERROR_PX = 4.0
TRI_MIN_ANGLE_DEG = 1.0


def triangulate_batch(K, R, t, ptr, cam, pix, *, max_error=TRI_MAX_ERROR_PX,
                      min_angle_deg=TRI_MIN_ANGLE_DEG, device=None, stream=None):
    """Cameras K/R/t (C,3,3)/(C,3,3)/(C,3); tracks as CSR (ptr, cam, pix).
    Returns (status, X, err): status 1 ok, 0 rejected, -1 degenerate, -2 too short."""
    import torch

    lib = _lib.load()
    dev = torch.device(device or "cuda")
    T = len(ptr) - 1

    def up(a, dt):
        a = np.ascontiguousarray(np.asarray(a, dtype=dt))
        if a.size == 0:
            a = np.zeros(1, dt)
        return torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)

    dK, dR, dt_ = up(np.reshape(K, (-1, 9)), np.float64), up(np.reshape(R, (-1, 9)), np.float64), \
        up(np.reshape(t, (-1, 3)), np.float64)
    dptr, dcam, dpix = up(ptr, np.int64), up(cam, np.int32), up(np.reshape(pix, (-1, 2)), np.float64)
    X = torch.empty((max(T, 1), 3), dtype=torch.float64, device=dev)
    err = torch.empty(max(T, 1), dtype=torch.float64, device=dev)
    status = torch.empty(max(T, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.msfm_triangulate_batch(_lib.ptr(dK), _lib.ptr(dR), _lib.ptr(dt_), T,
                                          _lib.ptr(dptr), _lib.ptr(dcam), _lib.ptr(dpix),
                                          float(max_error), float(min_angle_deg), _lib.ptr(X),
                                          _lib.ptr(err), _lib.ptr(status),
                                          _lib.stream_handle(stream)), "msfm_triangulate_batch")
    return status[:T].cpu().numpy(), X[:T].cpu().numpy(), err[:T].cpu().numpy()


def triangulate_track(observations, *, max_error=TRI_MAX_ERROR_PX,
                      min_angle_deg=TRI_MIN_ANGLE_DEG):
    """Drop-in for geometry.triangulate_track: Triangulated(point, mean_error) or
    None; InsufficientDataError / DegenerateGeometryError as the reference raises."""
    obs = list(observations)
    if len(obs) < 2:
        raise InsufficientDataError("need >= 2 observations")
    K = np.stack([np.asarray(c.K, np.float64) for c, _ in obs])
    R = np.stack([np.asarray(c.R, np.float64) for c, _ in obs])
    t = np.stack([np.asarray(c.t, np.float64).reshape(3) for c, _ in obs])
    pix = np.stack([np.asarray(p, np.float64).reshape(2) for _, p in obs])
    st, X, err = triangulate_batch(K, R, t, [0, len(obs)], np.arange(len(obs)), pix,
                                   max_error=max_error, min_angle_deg=min_angle_deg)
    if st[0] == -1:
        raise DegenerateGeometryError("triangulation rays are parallel or share one centre")
    if st[0] != 1:
        return None
    return Triangulated(point=X[0].copy(), mean_error=float(err[0]))
