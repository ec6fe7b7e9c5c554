"""Two-view geometry kept on the host, plus the triangulation drop-in.

``fundamental_from_poses`` is the reference's 3x3 float64 computation
(geometry.py:52-83), done with the same numpy operations so F is
bit-identical; it is 9 doubles per pair and never worth a kernel launch.
``triangulate_track`` / ``triangulate_batch`` (the K11 kernel) live in
``triangulation.py``.
"""

from __future__ import annotations

import numpy as np

from .types import DegenerateGeometryError, TwoViewGeometry


def _skew(v: np.ndarray) -> np.ndarray:
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def _canonical(F: np.ndarray) -> np.ndarray:
    """Frobenius normalisation, largest-magnitude entry positive (geometry.py:60-66)."""
    F = F / np.linalg.norm(F)
    if F.flat[np.abs(F).argmax()] < 0:
        F = -F
    return F


def fundamental_from_poses(cam_q, cam_c) -> TwoViewGeometry:
    """p_c^T F p_q = 0 for pose-known cameras (geometry.py:69-83)."""
    cq, cc = cam_q.center(), cam_c.center()
    baseline = cq - cc
    scale = max(np.linalg.norm(cq), np.linalg.norm(cc), 1.0)
    if np.linalg.norm(baseline) < 1e-12 * scale:
        raise DegenerateGeometryError(
            f"cameras {cam_q.image_id} and {cam_c.image_id} share a centre")
    F = np.linalg.inv(cam_c.K).T @ cam_c.R @ _skew(baseline) @ cam_q.R.T @ np.linalg.inv(cam_q.K)
    return TwoViewGeometry(F=_canonical(F), source="from_poses")
