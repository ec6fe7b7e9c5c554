"""ctypes binding of libmsfm_b200.so (the C-ABI in include/msfm_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises DeviceUnavailableError.
"""

from __future__ import annotations

import ctypes
import os

from .types import DeviceUnavailableError

_HERE = os.path.dirname(os.path.abspath(__file__))
# MSFM_B200_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("MSFM_B200_LIB") or os.path.join(_HERE, "libmsfm_b200.so")

c_int32_p = ctypes.POINTER(ctypes.c_int32)
VP = ctypes.c_void_p


class Bank(ctypes.Structure):
    _fields_ = [("d_xy", VP), ("d_desc", VP), ("d_norm2", VP), ("d_img_off", VP),
                ("d_img_n", VP), ("d_img_wh", VP), ("n_images", ctypes.c_int32),
                ("n_total", ctypes.c_int64)]


class Grids(ctypes.Structure):
    _fields_ = [("d_sub", VP), ("d_dims", VP), ("d_roff", VP), ("d_coff", VP),
                ("d_rstart", VP), ("d_cstart", VP), ("d_rmem", VP), ("d_cmem", VP),
                ("d_rrec", VP), ("d_crec", VP), ("D", ctypes.c_double)]


class MsftInfo(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("magic", ctypes.c_char * 4),
                ("version", ctypes.c_uint32), ("image_id", ctypes.c_int32),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("count", ctypes.c_int64), ("file_bytes", ctypes.c_int64),
                ("bad_record", ctypes.c_int64), ("bad_x", ctypes.c_float),
                ("bad_y", ctypes.c_float), ("bad_scale", ctypes.c_float)]


class ModelInfo(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("line", ctypes.c_int32),
                ("message", ctypes.c_char * 192), ("value", ctypes.c_double),
                ("value_id", ctypes.c_int64), ("n_cams", ctypes.c_int64),
                ("n_points", ctypes.c_int64), ("n_obs", ctypes.c_int64),
                ("stage", ctypes.c_char * 128), ("stage_truncated", ctypes.c_int32)]


class MatchParams(ctypes.Structure):
    _fields_ = [("d", ctypes.c_double), ("ratio", ctypes.c_float),
                ("single_cap", ctypes.c_float), ("max_nt", ctypes.c_int32),
                ("chunk_pairs", ctypes.c_int32), ("strategy", ctypes.c_int32),
                ("first_chunk_pairs", ctypes.c_int32),
                ("max_workspace_bytes", ctypes.c_int64)]


class StagePlan(ctypes.Structure):
    _fields_ = [("n_ranges", ctypes.c_int32), ("chunk", VP), ("img0", VP), ("img1", VP),
                ("bucket0", VP), ("bucket1", VP), ("feat0", VP), ("feat1", VP),
                ("landed", VP), ("n_buckets_total", ctypes.c_int64),
                ("grid_workspace", VP), ("grid_workspace_bytes", ctypes.c_size_t)]


_SIGS = {
    "msfm_last_error": (ctypes.c_char_p, []),
    "msfm_version": (ctypes.c_int, []),
    "msfm_launch_count": (ctypes.c_int64, []),
    "msfm_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "msfm_debug_counters": (ctypes.c_int, [ctypes.c_int, VP]),
    "msfm_profile_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_int64)]),
    "msfm_feature_norms": (ctypes.c_int, [VP, ctypes.c_int64, VP, VP]),
    "msfm_grid_dims": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, c_int32_p]),
    "msfm_grid_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64]),
    "msfm_grid_build": (ctypes.c_int, [ctypes.POINTER(Bank), VP, VP, VP, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_double, VP, VP, VP, VP, VP,
                                       VP, VP, VP, ctypes.c_size_t, VP]),
    "msfm_grid_build_range": (ctypes.c_int, [ctypes.POINTER(Bank), VP, VP, VP, ctypes.c_int64,
                                             ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.c_double, VP,
                                             VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP]),
    "msfm_guided_chunk_bounds": (ctypes.c_int32, [ctypes.c_int32, VP, ctypes.POINTER(MatchParams),
                                                  VP, ctypes.c_int32]),
    "msfm_ransac_samples": (ctypes.c_int, [VP, ctypes.c_int32, ctypes.c_uint32, ctypes.c_int64,
                                           ctypes.c_int32, ctypes.c_int32, VP, VP]),
    "msfm_model_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ModelInfo), VP, VP, VP, VP,
                                       VP, VP, VP, VP, VP, VP, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64]),
    "msfm_msft_load": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(MsftInfo), VP, VP, VP, VP,
                                      ctypes.c_int64]),
    "msfm_msft_load_many": (ctypes.c_int, [ctypes.c_int32, VP, VP, VP, VP, VP, VP, VP,
                                           ctypes.c_int32]),
    "msfm_ransac_samples_seeded_device": (ctypes.c_int, [ctypes.c_int32, VP, VP, ctypes.c_int32,
                                                         ctypes.c_int32, VP, VP, VP, VP]),
    "msfm_rng_seed_state": (ctypes.c_int, [ctypes.c_uint64, VP]),
    "msfm_ransac_samples_seeded": (ctypes.c_int, [ctypes.c_int32, VP, VP, ctypes.c_int32,
                                                  ctypes.c_int32, VP, VP]),
    "msfm_knn_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    "msfm_knn2_tracks": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.c_int32, VP, VP, ctypes.c_int32,
                                        VP, ctypes.c_int32, ctypes.c_int32, VP, VP, VP, VP,
                                        ctypes.c_size_t, VP]),
    "msfm_knn2_second_index": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.c_int32, VP, VP,
                                              ctypes.c_int32, VP, VP, VP, VP, VP, VP]),
    "msfm_track_sums": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.c_int64, VP, VP, VP, VP, VP,
                                       VP]),
    "msfm_knn2_float": (ctypes.c_int, [VP, ctypes.c_int64, VP, ctypes.c_int64, ctypes.c_int32,
                                       VP, VP, VP]),
    "msfm_gather_3d2d": (ctypes.c_int, [VP, VP, ctypes.c_int32, ctypes.c_int32, VP, VP, VP, VP,
                                        VP, VP, VP, VP]),
    "msfm_direct_3d2d": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.c_int32, VP, VP, ctypes.c_int32,
                                        VP, VP, VP, VP, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_double, VP, VP, VP, VP, VP, VP]),
    "msfm_pnp_hypotheses": (ctypes.c_int, [VP, VP, VP, VP, ctypes.c_int32, VP, ctypes.c_int32,
                                           ctypes.c_double, VP, VP, VP]),
    "msfm_pnp_refit": (ctypes.c_int, [VP, VP, VP, VP, ctypes.c_int32, VP, VP, ctypes.c_double,
                                      ctypes.c_int32, ctypes.c_int32, VP, VP, VP, VP, VP, VP]),
    "msfm_triangulate_batch": (ctypes.c_int, [VP, VP, VP, ctypes.c_int32, VP, VP, VP,
                                              ctypes.c_double, ctypes.c_double, VP, VP, VP, VP]),
    "msfm_fundamental_hypotheses": (ctypes.c_int, [VP, VP, VP, ctypes.c_int32, VP, ctypes.c_int32,
                                                   ctypes.c_double, VP, VP, VP]),
    "msfm_fundamental_refit": (ctypes.c_int, [VP, VP, VP, ctypes.c_int32, VP, VP, ctypes.c_double,
                                              VP, VP, VP, VP, VP]),
"msfm_covisibility": (ctypes.c_int, [ctypes.c_int32, VP, VP, ctypes.c_int32, VP, VP]),
    "msfm_merge_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int64]),
    "msfm_merge_tracks": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.c_int64, VP, VP, VP,
                                         ctypes.c_int32, VP, VP, VP, VP, VP, VP, VP,
                                         ctypes.c_size_t, VP]),
    "msfm_pack_matches": (ctypes.c_int, [ctypes.c_int32, VP, VP, VP, VP, VP, VP, VP, VP, VP]),
    "msfm_guided_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, VP,
                                                      ctypes.POINTER(MatchParams)]),
    "msfm_guided_match_rows": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.POINTER(Grids),
                                              ctypes.c_int32, VP, VP, VP, VP, VP, VP, VP,
                                              ctypes.POINTER(MatchParams), VP, VP, VP, VP, VP,
                                              VP, VP, VP, VP, VP, VP, VP, ctypes.c_size_t, VP, VP,
                                              ctypes.POINTER(StagePlan)]),
    "msfm_guided_match": (ctypes.c_int, [ctypes.POINTER(Bank), ctypes.POINTER(Grids),
                                         ctypes.c_int32, VP, VP, VP, VP, VP, VP, VP,
                                         ctypes.POINTER(MatchParams), VP, VP, VP, VP, VP, VP,
                                         VP, ctypes.c_size_t, VP]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(require_device: bool = True):
    """Load the library (and check a CUDA device exists unless told not to)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailableError(
                f"{LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise DeviceUnavailableError("no CUDA device visible: the B200 path has no CPU fallback")
    return _lib


class MsfmCallError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.msfm_last_error().decode(errors="replace") if _lib else ""
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise MsfmCallError(f"{what} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def h2d(a, dev):
    """A small host array on the device through pinned memory, asynchronously
    (a pageable copy would block the host until the stream drains)."""
    import numpy as np
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(dev, non_blocking=True)


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def launch_count() -> int:
    return int(load(require_device=False).msfm_launch_count())


def profile_enable(on: bool) -> None:
    check(load(require_device=False).msfm_profile_enable(1 if on else 0), "msfm_profile_enable")


def profile_read(name: str):
    """(total_ms, launches) of a library kernel recorded since profile_enable(True)."""
    ms = ctypes.c_double(0.0)
    n = ctypes.c_int64(0)
    check(load(require_device=False).msfm_profile_read(name.encode(), ctypes.byref(ms),
                                                         ctypes.byref(n)), "msfm_profile_read")
    return ms.value, n.value
