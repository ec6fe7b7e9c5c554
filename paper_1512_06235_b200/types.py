"""Host-side value types of the fine-stage path.

These mirror the data the reference stages hand to the hot path
(``msfm.features.FeatureSet`` features.py:44-96, ``msfm.model`` model.py:18-201,
``msfm.matching.Match`` matching.py:38-43, ``msfm.geometry`` geometry.py:28-49,
``msfm.descriptors.SearchStats`` descriptors.py:23-32, ``msfm.errors``).
The reference package is not present on the GPU box, so the drop-in carries
its own copies.  Every entry point in this package is duck-typed: objects of
the reference's own classes (same attribute names) are accepted unchanged,
which is what makes the package a drop-in for a running ``msfm`` pipeline.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import NamedTuple

import numpy as np

DESCRIPTOR_DIM = 128


# --------------------------------------------------------------------------
# errors (errors.py:4-42): same class names so callers' except-clauses read alike
# --------------------------------------------------------------------------

class MsfmError(Exception):
    pass


class FormatError(MsfmError):
    """Malformed input file (errors.py:12-13)."""


class DegenerateGeometryError(MsfmError):
    pass


class InsufficientDataError(MsfmError):
    pass


class NotRegisteredError(MsfmError):
    pass


class AlreadyRegisteredError(MsfmError):
    pass


class DeviceUnavailableError(MsfmError, RuntimeError):
    """The CUDA library is missing or no B200 is visible.  There is no CPU
    fallback: the product path fails loudly instead."""


# --------------------------------------------------------------------------
# features
# --------------------------------------------------------------------------

@dataclass
class FeatureSet:
    """One image's features, descending scale order (features.py:44-77)."""

    image_id: int
    width: int
    height: int
    xy: np.ndarray           # (n, 2) float32
    scale: np.ndarray        # (n,) float32
    orientation: np.ndarray  # (n,) float32
    descriptors: np.ndarray  # (n, 128) uint8
    coarse_count: int = -1
    _desc_f32: np.ndarray | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.coarse_count < 0:
            self.coarse_count = len(self.scale)

    def __len__(self) -> int:
        return len(self.scale)

    @property
    def tier_indices(self) -> np.ndarray:
        return np.arange(self.coarse_count)

    def descriptors_f32(self) -> np.ndarray:
        if self._desc_f32 is None:
            self._desc_f32 = np.ascontiguousarray(self.descriptors, dtype=np.float32)
        return self._desc_f32

    @classmethod
    def from_arrays(cls, image_id, width, height, xy, scale, orientation, descriptors):
        scale = np.asarray(scale, dtype=np.float32).reshape(-1)
        order = np.argsort(-scale, kind="stable")
        return cls(image_id=int(image_id), width=int(width), height=int(height),
                   xy=np.ascontiguousarray(np.asarray(xy, np.float32).reshape(-1, 2)[order]),
                   scale=np.ascontiguousarray(scale[order]),
                   orientation=np.ascontiguousarray(
                       np.asarray(orientation, np.float32).reshape(-1)[order]),
                   descriptors=np.ascontiguousarray(
                       np.asarray(descriptors, np.uint8).reshape(-1, DESCRIPTOR_DIM)[order]))


def select_top_scale(fs, eta: float = 20.0):
    """Coarse-tier boundary at the top eta percent (features.py:149-161)."""
    if not 0 < eta <= 100:
        raise ValueError(f"eta must be in (0, 100], got {eta}")
    n = len(fs)
    count = n if n < 1000 else int(np.ceil(eta / 100.0 * n))
    return replace(fs, coarse_count=count)


class FeatureStore:
    """image id -> FeatureSet (features.py:182-220)."""

    def __init__(self, sets=None):
        self.sets = dict(sets) if sets else {}

    def apply_eta(self, eta: float) -> None:
        for i in list(self.sets):
            self.sets[i] = select_top_scale(self.sets[i], eta)

    def image_ids(self):
        return sorted(self.sets)

    def __len__(self):
        return len(self.sets)

    def __getitem__(self, image_id):
        return self.sets[image_id]

    def __contains__(self, image_id):
        return image_id in self.sets

    def position(self, image_id, feature_id):
        return self.sets[image_id].xy[feature_id]

    def descriptor(self, image_id, feature_id):
        return self.sets[image_id].descriptors[feature_id]


# --------------------------------------------------------------------------
# model
# --------------------------------------------------------------------------

@dataclass(frozen=True, order=True)
class FeatureRef:
    image_id: int
    feature_id: int


@dataclass
class Camera:
    """x ~ K (R X + t) (model.py:26-53)."""

    K: np.ndarray
    R: np.ndarray
    t: np.ndarray
    image_id: int

    def __post_init__(self):
        self.K = np.asarray(self.K, dtype=np.float64).reshape(3, 3)
        self.R = np.asarray(self.R, dtype=np.float64).reshape(3, 3)
        self.t = np.asarray(self.t, dtype=np.float64).reshape(3)

    def center(self) -> np.ndarray:
        return -self.R.T @ self.t

    def project(self, X):
        X = np.asarray(X, dtype=np.float64).reshape(-1, 3)
        xc = X @ self.R.T + self.t
        uv = xc @ self.K.T
        return uv[:, :2] / uv[:, 2:3], xc[:, 2]


def make_intrinsics(focal: float, cx: float, cy: float) -> np.ndarray:
    return np.array([[focal, 0.0, cx], [0.0, focal, cy], [0.0, 0.0, 1.0]])


@dataclass
class Point3D:
    position: np.ndarray
    track: dict = field(default_factory=dict)  # image_id -> feature_id
    mean_descriptor: np.ndarray | None = None

    def refs(self):
        return [FeatureRef(i, f) for i, f in sorted(self.track.items())]

    def track_length(self) -> int:
        return len(self.track)


class Model:
    """Cameras + points with owner/visibility indexes (model.py:75-201)."""

    def __init__(self, stage_tag: str = ""):
        self.cameras: dict[int, Camera] = {}
        self.points: dict[int, Point3D] = {}
        self.stage_tag = stage_tag
        self._next_point_id = 0
        self._owner: dict[FeatureRef, int] = {}
        self._visible: dict[int, set] = {}

    def is_registered(self, image_id):
        return image_id in self.cameras

    def image_ids(self):
        return sorted(self.cameras)

    def point_ids(self):
        return sorted(self.points)

    def owner(self, ref):
        return self._owner.get(ref)

    def points_visible_in(self, image_id):
        if image_id not in self.cameras:
            raise NotRegisteredError(f"image {image_id} is not registered")
        return set(self._visible.get(image_id, ()))

    def covisible_points(self, a, b):
        for i in (a, b):
            if i not in self.cameras:
                raise NotRegisteredError(f"image {i} is not registered")
        return self._visible.get(a, set()) & self._visible.get(b, set())

    def attach_camera(self, camera, inliers=()) -> int:
        iid = camera.image_id
        if iid in self.cameras:
            raise AlreadyRegisteredError(f"image {iid} already registered")
        inliers = list(inliers)
        for pid, ref in inliers:
            if pid not in self.points:
                raise KeyError(f"unknown point id {pid}")
            if ref.image_id != iid:
                raise ValueError(f"{ref} does not belong to image {iid}")
        self.cameras[iid] = camera
        self._visible.setdefault(iid, set())
        dropped = 0
        for pid, ref in inliers:
            if ref in self._owner or iid in self.points[pid].track:
                dropped += 1
            else:
                self._link(pid, ref)
        return dropped

    def add_point(self, position, refs) -> int:
        refs = list(refs)
        if len(refs) < 2 or len({r.image_id for r in refs}) < len(refs):
            raise ValueError("a track needs >= 2 features from distinct images")
        for r in refs:
            if r.image_id not in self.cameras:
                raise NotRegisteredError(f"image {r.image_id} is not registered")
            if r in self._owner:
                raise ValueError(f"{r} already belongs to point {self._owner[r]}")
        pid = self._next_point_id
        self._next_point_id += 1
        self.points[pid] = Point3D(position=np.asarray(position, np.float64).copy())
        for r in refs:
            self._link(pid, r)
        return pid

    def extend_track(self, pid, ref) -> bool:
        if ref.image_id not in self.cameras:
            raise NotRegisteredError(f"image {ref.image_id} is not registered")
        if ref in self._owner or ref.image_id in self.points[pid].track:
            return False
        self._link(pid, ref)
        return True

    def set_position(self, pid, position):
        self.points[pid].position = np.asarray(position, np.float64).copy()

    def _link(self, pid, ref):
        self.points[pid].track[ref.image_id] = ref.feature_id
        self.points[pid].mean_descriptor = None
        self._owner[ref] = pid
        self._visible.setdefault(ref.image_id, set()).add(pid)


# --------------------------------------------------------------------------
# matching / geometry results
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Match:
    query: FeatureRef
    target: FeatureRef
    distance: float
    ratio: float


@dataclass
class TwoViewGeometry:
    F: np.ndarray
    inlier_count: int = 0
    source: str = "estimated"
    degenerate_planar: bool = False


@dataclass
class Edge:
    """matching.py:46-56"""
    matches: list
    geometry: TwoViewGeometry | None = None
    inlier_mask: np.ndarray | None = None

    def inlier_matches(self) -> list:
        if self.inlier_mask is None:
            return list(self.matches)
        return [m for m, keep in zip(self.matches, self.inlier_mask) if keep]


@dataclass
class MatchGraph:
    """matching.py:59-79"""
    edges: dict = field(default_factory=dict)

    def pair_key(self, a: int, b: int):
        return (a, b) if a < b else (b, a)

    def get(self, a: int, b: int):
        return self.edges.get(self.pair_key(a, b))

    def neighbors(self, image_id: int) -> list:
        out = []
        for a, b in self.edges:
            if a == image_id:
                out.append(b)
            elif b == image_id:
                out.append(a)
        return sorted(out)

    def match_count(self, a: int, b: int) -> int:
        edge = self.get(a, b)
        return len(edge.matches) if edge else 0


@dataclass(frozen=True)
class EpipolarLine:
    a: float
    b: float
    c: float


class Triangulated(NamedTuple):
    point: np.ndarray
    mean_error: float


@dataclass
class SearchStats:
    queries: int = 0
    candidates: int = 0

    def add(self, queries: int, candidates: int) -> None:
        self.queries += queries
        self.candidates += candidates



@dataclass
class LocalizationResult:
    """localize.py:41-48"""
    image_id: int
    method: str
    correspondences: list = field(default_factory=list)
    pose: object = None
    inliers: int = 0
    inlier_refs: list = field(default_factory=list)
    reason: str = ""


@dataclass
class SetCover:
    """localize.py:34-38"""
    selected: list
    k: int
    coverage: dict


# --------------------------------------------------------------------------
# the caller's own classes (SURVEY.md §8b "Data crossing" / "Error conventions")
# --------------------------------------------------------------------------
# When the reference package ``msfm`` is importable, every value type and error
# class above is replaced by the reference's own class, in this module and in
# every module of the package that bound it, so a drop-in raises
# ``msfm.errors.InsufficientDataError`` and returns ``msfm.matching.Match`` /
# ``msfm.model.FeatureRef`` objects that compare, hash and sort with the
# caller's.  On a box without ``msfm`` (the GPU pool) the classes above stand in.

_REFERENCE_CLASSES = {
    "MsfmError": ("msfm.errors", "MsfmError"),
    "FormatError": ("msfm.errors", "FormatError"),
    "DegenerateGeometryError": ("msfm.errors", "DegenerateGeometryError"),
    "InsufficientDataError": ("msfm.errors", "InsufficientDataError"),
    "NotRegisteredError": ("msfm.errors", "NotRegisteredError"),
    "AlreadyRegisteredError": ("msfm.errors", "AlreadyRegisteredError"),
    "FeatureSet": ("msfm.features", "FeatureSet"),
    "FeatureStore": ("msfm.features", "FeatureStore"),
    "FeatureRef": ("msfm.model", "FeatureRef"),
    "Camera": ("msfm.model", "Camera"),
    "Point3D": ("msfm.model", "Point3D"),
    "Model": ("msfm.model", "Model"),
    "Match": ("msfm.matching", "Match"),
    "Edge": ("msfm.matching", "Edge"),
    "MatchGraph": ("msfm.matching", "MatchGraph"),
    "TwoViewGeometry": ("msfm.geometry", "TwoViewGeometry"),
    "EpipolarLine": ("msfm.geometry", "EpipolarLine"),
    "Triangulated": ("msfm.geometry", "Triangulated"),
    "SearchStats": ("msfm.descriptors", "SearchStats"),
    "LocalizationResult": ("msfm.localize", "LocalizationResult"),
    "SetCover": ("msfm.localize", "SetCover"),
}
_LOCAL_CLASSES: dict = {}
REFERENCE_TYPES = False


def reference_available() -> bool:
    import importlib.util

    try:
        return importlib.util.find_spec("msfm") is not None
    except (ImportError, ValueError):
        return False


def adopt_reference_types() -> bool:
    """Rebind the package's value types and errors to ``msfm``'s classes (idempotent).
    Returns True when the reference classes are in use."""
    global REFERENCE_TYPES, DeviceUnavailableError
    import importlib
    import sys

    if REFERENCE_TYPES:
        return True
    if not reference_available():
        return False
    g = globals()
    local = {}
    ref = {}
    for name, (mod, attr) in _REFERENCE_CLASSES.items():
        try:
            cls = getattr(importlib.import_module(mod), attr)
        except (ImportError, AttributeError):
            continue
        ref[name] = cls
    if "MsfmError" not in ref:
        return False
    for name in ref:
        if name in g:
            local[name] = g[name]
    # the device error keeps its name but joins the reference hierarchy
    old_dev = DeviceUnavailableError
    DeviceUnavailableError = type("DeviceUnavailableError", (ref["MsfmError"], RuntimeError),
                                  {"__doc__": old_dev.__doc__, "__module__": __name__})
    local["DeviceUnavailableError"] = old_dev
    ref["DeviceUnavailableError"] = DeviceUnavailableError
    pkg = __name__.rsplit(".", 1)[0]
    for mname, m in list(sys.modules.items()):
        if m is None or not (mname == pkg or mname.startswith(pkg + ".")):
            continue
        d = vars(m)
        for key, val in list(d.items()):
            for name, old in local.items():
                if val is old and name in ref:
                    d[key] = ref[name]
    _LOCAL_CLASSES.update(local)
    REFERENCE_TYPES = True
    return True
