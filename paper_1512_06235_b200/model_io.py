"""Model snapshots (.msfm text, msfm.io io.py:16-84) read natively into the CSR
arrays the device stages consume, and the ``read_model`` drop-in on top of them.

``read_snapshot`` is the throughput path: one pass of C++ (``msfm_model_read``,
csrc/model_io.cpp) validates the file in the reference's order and fills flat
arrays — cameras (id, K, R, t) and points (xyz, track CSR in file order) — with no
per-record Python.  ``read_model`` builds the reference's ``Model`` from those
arrays and raises the reference's ``FormatError`` messages.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class ModelArrays:
    """A model snapshot as arrays; point ids are the record order (0..n-1)."""

    stage_tag: str
    cam_id: np.ndarray          # (C,) int32, file order
    K: np.ndarray               # (C, 3, 3) f64 (make_intrinsics(f, cx, cy))
    R: np.ndarray               # (C, 3, 3) f64
    t: np.ndarray               # (C, 3) f64
    point_xyz: np.ndarray       # (P, 3) f64
    track_ptr: np.ndarray       # (P+1,) int64
    track_img: np.ndarray       # (obs,) int32
    track_fid: np.ndarray       # (obs,) int32


def _format_error():
    from . import types
    return types.FormatError


def _raise_for(path, info):
    FormatError = _format_error()
    st = info.status
    msg = info.message.decode(errors="replace")
    if st == 6:
        open(path, "rb").close()                         # the native OSError
        raise OSError(f"{path}: unreadable")
    if st == 1:
        raise FormatError(f"{path}: {msg}")
    if st == 4:
        raise FormatError(f"{path}:{info.line}: camera {info.value_id}: det(R) = "
                          f"{np.float64(info.value)}")
    if st == 7:
        raise OSError(f"{path}: changed while loading")
    raise FormatError(f"{path}:{info.line}: {msg}")


def read_snapshot(path) -> ModelArrays:
    """Parse and validate a model file natively (io.py:51-84 semantics)."""
    lib = _lib.load(require_device=False)
    info = _lib.ModelInfo()
    bpath = os.fsencode(str(path))
    null = [None] * 10
    lib.msfm_model_read(bpath, ctypes.byref(info), *null, 0, 0, 0)
    if info.status != 0:
        _raise_for(path, info)
    C, P, O = int(info.n_cams), int(info.n_points), int(info.n_obs)
    cam_id = np.zeros(max(C, 1), np.int32)
    fcc = np.zeros((max(C, 1), 3))
    R = np.zeros((max(C, 1), 3, 3))
    t = np.zeros((max(C, 1), 3))
    cline = np.zeros(max(C, 1), np.int32)
    xyz = np.zeros((max(P, 1), 3))
    ptr = np.zeros(P + 1, np.int64)
    timg = np.zeros(max(O, 1), np.int32)
    tfid = np.zeros(max(O, 1), np.int32)
    pline = np.zeros(max(P, 1), np.int32)
    p = lambda a: a.ctypes.data
    lib.msfm_model_read(bpath, ctypes.byref(info), p(cam_id), p(fcc), p(R), p(t), p(cline),
                        p(xyz), p(ptr), p(timg), p(tfid), p(pline), C, P, O)
    if info.status != 0:
        _raise_for(path, info)
    K = np.zeros((C, 3, 3))
    K[:, 0, 0] = fcc[:C, 0]
    K[:, 1, 1] = fcc[:C, 0]
    K[:, 0, 2] = fcc[:C, 1]
    K[:, 1, 2] = fcc[:C, 2]
    K[:, 2, 2] = 1.0
    stage = info.stage.decode()
    if info.stage_truncated:                 # rare: tags longer than the native buffer
        with open(path) as f:
            for line in f.read().splitlines()[1:]:
                fields = line.split()
                if fields and fields[0] == "STAGE":
                    stage = fields[1] if len(fields) > 1 else ""
    return ModelArrays(stage_tag=stage, cam_id=cam_id[:C], K=K, R=R[:C], t=t[:C],
                       point_xyz=xyz[:P], track_ptr=ptr, track_img=timg[:O], track_fid=tfid[:O])


def read_model(path):
    """Drop-in for msfm.io.read_model (io.py:51-84): a Model (the reference's class
    when it is importable) from the natively parsed arrays."""
    from . import types

    arr = read_snapshot(path)
    model = types.Model(stage_tag=arr.stage_tag)
    for k in range(len(arr.cam_id)):
        model.attach_camera(types.Camera(K=arr.K[k], R=arr.R[k], t=arr.t[k],
                                         image_id=int(arr.cam_id[k])))
    FR = types.FeatureRef
    img, fid, ptr = arr.track_img.tolist(), arr.track_fid.tolist(), arr.track_ptr.tolist()
    for q in range(len(arr.point_xyz)):
        a, b = ptr[q], ptr[q + 1]
        model.add_point(arr.point_xyz[q], [FR(i, f) for i, f in zip(img[a:b], fid[a:b])])
    return model
