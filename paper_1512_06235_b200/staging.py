"""Feature-file staging (features.py:98-130, 182-198) through the native loader.

``load_features`` / ``load_dir`` are drop-ins for the reference's readers (same
validation order and FormatError messages); ``host_bank_from_dir`` reads a whole
directory of ``.msft`` files on host threads straight into the pinned host bank
the device path uploads from, with no per-record Python work.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _lib

HEADER_BYTES = 24
RECORD_BYTES = 144


def _errors():
    try:
        from msfm.errors import FormatError
        return FormatError
    except Exception:
        from .types import FormatError
        return FormatError


def _feature_set_type():
    try:
        from msfm.features import FeatureSet
        return FeatureSet
    except Exception:
        from .types import FeatureSet
        return FeatureSet


def _raise_for(path, info):
    """The reference's FormatError for a failed file (features.py:101-125)."""
    FormatError = _errors()
    st = info.status
    if st == 6:
        open(path, "rb").close()                      # raise the native OSError
        raise OSError(f"{path}: unreadable")
    if st == 7:
        # only a file rewritten between the size probe and the read gets here (the
        # reference reads once); nothing was written to the caller's buffers
        raise OSError(f"{path}: changed while loading ({info.count} records, sized for fewer/more)")
    if st == 1:
        raise FormatError(f"{path}: truncated header, file ends at byte {info.file_bytes}")
    if st == 2:
        raise FormatError(f"{path}: bad magic {bytes(info.magic)!r} at byte 0")
    if st == 3:
        raise FormatError(f"{path}: unsupported version {info.version} at byte 4")
    if st == 4:
        expected = HEADER_BYTES + info.count * RECORD_BYTES
        raise FormatError(f"{path}: payload ends at byte {info.file_bytes}, expected {expected} "
                          f"({info.count} records of {RECORD_BYTES} bytes)")
    if st == 5:
        i = info.bad_record
        raise FormatError(f"{path}: record {i} at byte {HEADER_BYTES + i * RECORD_BYTES} "
                          f"violates bounds (x={np.float32(info.bad_x)}, y={np.float32(info.bad_y)}, "
                          f"scale={np.float32(info.bad_scale)})")


def load_features(path):
    """Drop-in for msfm.features.load_features: a FeatureSet in descending-scale
    order, FormatError as the reference raises it."""
    lib = _lib.load(require_device=False)
    info = _lib.MsftInfo()
    bpath = os.fsencode(path)
    lib.msfm_msft_load(bpath, ctypes.byref(info), None, None, None, None, -1)
    if info.status != 0:
        _raise_for(path, info)
    n = int(info.count)
    xy = np.empty((n, 2), np.float32)
    scale = np.empty(n, np.float32)
    orient = np.empty(n, np.float32)
    desc = np.empty((n, 128), np.uint8)
    lib.msfm_msft_load(bpath, ctypes.byref(info), xy.ctypes.data, scale.ctypes.data,
                       orient.ctypes.data, desc.ctypes.data, n)
    if info.status != 0:
        _raise_for(path, info)
    return _feature_set_type()(image_id=int(info.image_id), width=int(info.width),
                               height=int(info.height), xy=xy, scale=scale, orientation=orient,
                               descriptors=desc)


def load_dir(directory, eta=None):
    """Drop-in for FeatureStore.load_dir (features.py:186-198)."""
    try:
        from msfm.features import FeatureStore
    except Exception:
        from .types import FeatureStore
    FormatError = _errors()
    store = FeatureStore()
    for path in sorted(Path(directory).glob("*.msft")):
        fs = load_features(path)
        if fs.image_id in store.sets:
            raise FormatError(f"{path}: duplicate image id {fs.image_id}")
        store.sets[fs.image_id] = fs
    if eta is not None:
        store.apply_eta(eta)
    return store


def host_bank_from_dir(directory, n_threads=None):
    """HostBank (pinned xy / descriptors, images in ascending id) read natively
    from every *.msft file of a directory."""
    import torch

    from .bank import HostBank

    lib = _lib.load(require_device=False)
    FormatError = _errors()
    paths = sorted(Path(directory).glob("*.msft"))
    infos = (_lib.MsftInfo * max(len(paths), 1))()
    for k, p in enumerate(paths):
        lib.msfm_msft_load(os.fsencode(p), ctypes.byref(infos[k]), None, None, None, None, -1)
        if infos[k].status != 0:
            _raise_for(p, infos[k])
    ids = [int(infos[k].image_id) for k in range(len(paths))]
    if len(set(ids)) != len(ids):
        seen = set()
        for p, i in zip(paths, ids):
            if i in seen:
                raise FormatError(f"{p}: duplicate image id {i}")
            seen.add(i)
    order = np.argsort(ids, kind="stable")
    counts = np.array([int(infos[k].count) for k in order], np.int64)
    off = np.zeros(len(order) + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    n = int(counts.sum())
    xy = torch.empty((max(n, 1), 2), dtype=torch.float32).pin_memory()
    desc = torch.empty((max(n, 1), 128), dtype=torch.uint8).pin_memory()
    cpaths = (ctypes.c_char_p * max(len(order), 1))(*[os.fsencode(paths[k]) for k in order])
    row_off = np.ascontiguousarray(off)
    out_infos = (_lib.MsftInfo * max(len(order), 1))()
    lib.msfm_msft_load_many(len(order), cpaths, row_off.ctypes.data, out_infos, xy.data_ptr(),
                            None, None, desc.data_ptr(), int(n_threads or os.cpu_count() or 1))
    for j, k in enumerate(order):
        if out_infos[j].status != 0:
            _raise_for(paths[k], out_infos[j])
    wh = np.array([[int(infos[k].width), int(infos[k].height)] for k in order], np.int64)
    return HostBank.from_buffers([ids[k] for k in order], counts, wh, xy[:n], desc[:n])
