"""Seeded synthetic scenes: the input generator for every benchmark config.

Restates ``msfm.synth.generate_scene`` (synth.py:197-292) with the identical
``np.random.default_rng(seed)`` draw order, so a scene generated here is the
same scene the reference generates (pinned by tests/test_synth_golden.py
against fixtures produced from the reference).  Nothing here is on the
measured path; it only manufactures inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .types import DESCRIPTOR_DIM, Camera, FeatureSet, FeatureStore, make_intrinsics

_LEVELS = 24  # synth.py:20


@dataclass
class SceneSpec:
    n_cameras: int = 20
    layout: str = "ring"
    n_points: int = 2000
    image_width: int = 1024
    image_height: int = 768
    focal: float = 900.0
    ring_radius: float = 6.0
    cloud_radius: float = 2.0
    pixel_noise: float = 0.0
    descriptor_noise: float = 0.0
    repetition_groups: int = 0
    repetition_group_size: int = 0
    visibility_fraction: float = 1.0
    clutter_per_image: int = 0
    seed: int = 0


@dataclass
class Scene:
    spec: SceneSpec
    cameras: list
    points: np.ndarray
    feature_sets: dict
    point_of_feature: dict  # image id -> (n,) int64 world point id, -1 clutter
    warnings: list = field(default_factory=list)

    def store(self) -> FeatureStore:
        return FeatureStore(self.feature_sets)

    def oracle_matches(self, a: int, b: int):
        ta, tb = self.point_of_feature[a], self.point_of_feature[b]
        pos_b = {int(p): j for j, p in enumerate(tb) if p >= 0}
        return [(i, pos_b[int(p)]) for i, p in enumerate(ta) if p >= 0 and int(p) in pos_b]


def _rig(spec: SceneSpec, rng) -> np.ndarray:
    """Camera centres (synth.py:142-167)."""
    n = spec.n_cameras
    if spec.layout == "ring":
        th = 2.0 * np.pi * np.arange(n) / n
        return np.stack([spec.ring_radius * np.cos(th), spec.ring_radius * np.sin(th),
                         0.3 * np.sin(3.0 * th)], axis=1)
    if spec.layout == "grid":
        side = int(np.ceil(np.sqrt(n)))
        gx, gy = np.meshgrid(np.arange(side), np.arange(side))
        cell = np.stack([gx.ravel(), gy.ravel()], axis=1)[:n].astype(np.float64)
        out = np.zeros((n, 3))
        denom = max(side - 1, 1)
        out[:, 0] = (cell[:, 0] / denom - 0.5) * spec.ring_radius
        out[:, 2] = (cell[:, 1] / denom - 0.5) * spec.ring_radius
        out[:, 1] = -spec.ring_radius
        return out
    if spec.layout == "sphere_cap":
        phi = rng.uniform(0.0, 2.0 * np.pi, size=n)
        z = rng.uniform(np.cos(np.pi / 3.0), 1.0, size=n)
        s = np.sqrt(1.0 - z ** 2)
        return spec.ring_radius * np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    raise ValueError(f"unknown layout {spec.layout!r}")


def _rotation_towards_origin(c: np.ndarray) -> np.ndarray:
    fwd = -c / np.linalg.norm(-c)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.98:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    return np.stack([right, np.cross(fwd, right), fwd])


def _levels(rng, n):
    w = 2.0 ** -np.arange(_LEVELS, dtype=np.float64)
    return rng.choice(_LEVELS, size=n, p=w / w.sum())


def generate_scene(spec: SceneSpec, first_cameras: int | None = None) -> Scene:
    """``first_cameras``: stop after that many cameras' feature sets.  The draws
    are sequential per camera, so those cameras (and every pose and point) are
    exactly the full scene's; used to sample the 3000-camera C5 recipe."""
    rng = np.random.default_rng(spec.seed)
    centres = _rig(spec, rng)
    K = make_intrinsics(spec.focal, spec.image_width / 2.0, spec.image_height / 2.0)
    cams = []
    for i in range(spec.n_cameras):
        R = _rotation_towards_origin(centres[i])
        cams.append(Camera(K=K, R=R, t=-R @ centres[i], image_id=i))

    X = rng.normal(size=(spec.n_points, 3))
    X /= np.maximum(np.linalg.norm(X, axis=1, keepdims=True), 1e-12)
    X *= spec.cloud_radius * rng.uniform(0.2, 1.0, size=(spec.n_points, 1)) ** (1.0 / 3.0)
    normals = X.copy()
    normals[np.linalg.norm(normals, axis=1) < 1e-9] = np.array([0.0, 0.0, 1.0])
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)

    n_rep = spec.repetition_groups * spec.repetition_group_size
    if n_rep > spec.n_points:
        raise ValueError("repetition groups exceed the point count")
    base = rng.integers(0, 256, size=(spec.n_points, DESCRIPTOR_DIM), dtype=np.uint8)
    for g in range(spec.repetition_groups):
        lo = g * spec.repetition_group_size
        base[lo:lo + spec.repetition_group_size] = base[lo]
    point_levels = _levels(rng, spec.n_points)
    cos_cone = np.cos(spec.visibility_fraction * np.pi)

    W, H = spec.image_width, spec.image_height
    sets, owners, warnings = {}, {}, []
    for cam in cams[:first_cameras]:
        uv, depth = cam.project(X)
        if spec.pixel_noise > 0:
            uv = uv + rng.normal(0.0, spec.pixel_noise, size=uv.shape)
        to_cam = cam.center()[None, :] - X
        to_cam /= np.maximum(np.linalg.norm(to_cam, axis=1, keepdims=True), 1e-12)
        seen = np.flatnonzero((np.einsum("ij,ij->i", normals, to_cam) >= cos_cone)
                              & (depth > 0.1) & (uv[:, 0] >= 0) & (uv[:, 0] < W)
                              & (uv[:, 1] >= 0) & (uv[:, 1] < H))
        if len(seen) < 8:
            warnings.append(f"camera {cam.image_id} sees only {len(seen)} points")
        nv, nc = len(seen), spec.clutter_per_image
        xy = np.zeros((nv + nc, 2))
        desc = np.zeros((nv + nc, DESCRIPTOR_DIM))
        pid = np.full(nv + nc, -1, dtype=np.int64)
        xy[:nv], desc[:nv], pid[:nv] = uv[seen], base[seen], seen
        lv = np.concatenate([point_levels[seen], _levels(rng, nc)])
        if nc:
            xy[nv:] = rng.uniform(0.0, [W - 1e-3, H - 1e-3], size=(nc, 2))
            desc[nv:] = rng.integers(0, 256, size=(nc, DESCRIPTOR_DIM))
        if spec.descriptor_noise > 0:
            desc = desc + rng.normal(0.0, spec.descriptor_noise, size=desc.shape)
        desc = np.clip(np.round(desc), 0, 255).astype(np.uint8)
        jit = rng.uniform(-0.45, 0.45, size=nv + nc)
        scale = (1.6 * 2.0 ** ((lv.astype(np.float64) + jit) / 3.0)).astype(np.float32)
        orient = rng.uniform(0.0, 2.0 * np.pi, size=nv + nc).astype(np.float32)
        order = np.argsort(-scale, kind="stable")
        sets[cam.image_id] = FeatureSet(
            image_id=cam.image_id, width=W, height=H,
            xy=np.ascontiguousarray(xy[order], dtype=np.float32),
            scale=np.ascontiguousarray(scale[order]),
            orientation=np.ascontiguousarray(orient[order]),
            descriptors=np.ascontiguousarray(desc[order]))
        owners[cam.image_id] = pid[order]
    return Scene(spec=spec, cameras=cams, points=X, feature_sets=sets,
                 point_of_feature=owners, warnings=warnings)
