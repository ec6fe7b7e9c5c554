"""Device-resident feature bank and spatial index.

All images of a stage live in HBM as one SoA: xy f32 (n,2), descriptors u8
(n,128) in 16-byte-aligned rows (so a 128-B row is eight coalesced 16-B
vector loads), |desc|^2 i32 (n), plus per-image offsets.  The target-image
index (build_grid, guided.py:110-137) is built once per stage on the device.
Host arrays are staged through pinned memory and copied with one
``cudaMemcpyAsync`` per array.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _slots(bank, image_ids) -> np.ndarray:
    ids = np.asarray(image_ids, dtype=np.int64).reshape(-1)
    if "_ids_sorted" not in bank.__dict__:
        keys = np.array(bank.image_ids, dtype=np.int64)
        order = np.argsort(keys, kind="stable")
        bank.__dict__["_ids_sorted"], bank.__dict__["_ids_order"] = keys[order], order
    srt, order = bank.__dict__["_ids_sorted"], bank.__dict__["_ids_order"]
    if len(ids) == 0:
        return np.zeros(0, np.int64)
    pos = np.searchsorted(srt, ids)
    pos_c = np.minimum(pos, max(len(srt) - 1, 0))
    bad = (pos >= len(srt)) | (srt[pos_c] != ids)
    if np.any(bad):
        raise KeyError(int(ids[np.flatnonzero(bad)[0]]))
    return order[pos_c].astype(np.int64)


class HostBank:
    """Concatenated feature arrays in pinned host memory (the H2D staging area)."""

    def slots(self, image_ids) -> np.ndarray:
        """Bank index of every image id (int64), KeyError for ids not in the bank."""
        return _slots(self, image_ids)

    def __init__(self, feature_sets, image_ids=None):
        import torch

        ids = sorted(feature_sets) if image_ids is None else list(image_ids)
        sets = [feature_sets[i] for i in ids]
        self.image_ids = ids
        self.counts = np.array([len(fs) for fs in sets], dtype=np.int64)
        self.offsets = np.zeros(len(sets), dtype=np.int64)
        if len(sets) > 1:
            np.cumsum(self.counts[:-1], out=self.offsets[1:])
        self.wh = np.array([[int(fs.width), int(fs.height)] for fs in sets],
                           dtype=np.int32).reshape(-1, 2)
        n = int(self.counts.sum())
        self.xy = torch.empty((n, 2), dtype=torch.float32).pin_memory()
        self.desc = torch.empty((n, 128), dtype=torch.uint8).pin_memory()
        xy_np, desc_np = self.xy.numpy(), self.desc.numpy()
        for k, fs in enumerate(sets):
            lo, hi = self.offsets[k], self.offsets[k] + self.counts[k]
            xy_np[lo:hi] = np.asarray(fs.xy, np.float32).reshape(-1, 2)
            desc_np[lo:hi] = np.asarray(fs.descriptors, np.uint8).reshape(-1, 128)
        self.img_off = torch.from_numpy(self.offsets.copy()).pin_memory()
        self.img_n = torch.from_numpy(self.counts.astype(np.int32)).pin_memory()
        self.img_wh = torch.from_numpy(self.wh.copy()).pin_memory()

    @classmethod
    def from_buffers(cls, image_ids, counts, wh, xy, desc):
        """A bank over already-filled pinned buffers (staging.host_bank_from_dir)."""
        import torch

        self = cls.__new__(cls)
        self.image_ids = list(image_ids)
        self.counts = np.asarray(counts, np.int64)
        self.offsets = np.zeros(len(self.counts), dtype=np.int64)
        if len(self.counts) > 1:
            np.cumsum(self.counts[:-1], out=self.offsets[1:])
        self.wh = np.asarray(wh, np.int32).reshape(-1, 2)
        self.xy, self.desc = xy, desc
        self.img_off = torch.from_numpy(self.offsets.copy()).pin_memory()
        self.img_n = torch.from_numpy(self.counts.astype(np.int32)).pin_memory()
        self.img_wh = torch.from_numpy(self.wh.copy()).pin_memory()
        return self

    @property
    def nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size())
                   for t in (self.xy, self.desc, self.img_off, self.img_n, self.img_wh))


class FeatureBank:
    """Feature sets of many images, resident on one CUDA device."""

    def __init__(self, feature_sets=None, device=None, image_ids=None, stream=None, host=None,
                 staged: bool = False):
        """``staged``: allocate the device rows without copying them; the caller
        fills image ranges with ``stage_range`` (and indexes them with
        ``SpatialIndex.build_range``) on streams of its choice."""
        import torch

        lib = _lib.load()
        self.device = torch.device(device or "cuda")
        if host is None:
            host = HostBank(feature_sets, image_ids)
        self.image_ids = host.image_ids
        self.index_of = {i: k for k, i in enumerate(self.image_ids)}
        self.counts, self.offsets, self.wh = host.counts, host.offsets, host.wh
        self.n_total = int(self.counts.sum())
        dev = self.device
        self.host = host
        if staged:
            self.xy = torch.empty(tuple(host.xy.shape), dtype=torch.float32, device=dev)
            self.desc = torch.empty(tuple(host.desc.shape), dtype=torch.uint8, device=dev)
        else:
            self.xy = host.xy.to(dev, non_blocking=True)
            self.desc = host.desc.to(dev, non_blocking=True)
        self.img_off = host.img_off.to(dev, non_blocking=True)
        self.img_n = host.img_n.to(dev, non_blocking=True)
        self.img_wh = host.img_wh.to(dev, non_blocking=True)
        self.norm2 = torch.empty(self.n_total, dtype=torch.int32, device=dev)
        self.staged = staged
        if not staged:
            st = _lib.stream_handle(stream)
            _lib.check(lib.msfm_feature_norms(_lib.ptr(self.desc), self.n_total,
                                              _lib.ptr(self.norm2), st), "msfm_feature_norms")
        self.max_n = int(self.counts.max()) if len(self.counts) else 0
        self._grids = {}

    def slots(self, image_ids) -> np.ndarray:
        """Bank index of every image id (int64), KeyError for ids not in the bank."""
        return _slots(self, image_ids)

    def refill(self, stream=None):
        """Copy every host row into this bank's device buffers again and recompute
        |desc|^2 (a step of a pipeline whose inputs arrive in the same pinned host
        bank: no device allocation).  Spatial indexes are dropped."""
        import torch

        lib = _lib.load()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            self.xy.copy_(self.host.xy, non_blocking=True)
            self.desc.copy_(self.host.desc, non_blocking=True)
        _lib.check(lib.msfm_feature_norms(_lib.ptr(self.desc), self.n_total, _lib.ptr(self.norm2),
                                          _lib.stream_handle(s)), "msfm_feature_norms")
        self._grids = {}

    def row_range(self, k0: int, k1: int):
        """Bank rows [a, b) of images [k0, k1)."""
        a = int(self.offsets[k0]) if k0 < len(self.offsets) else self.n_total
        b = int(self.offsets[k1]) if k1 < len(self.offsets) else self.n_total
        return a, b

    def upload_range(self, k0: int, k1: int, copy_stream):
        """(staged bank) Copy the rows of images [k0, k1) on ``copy_stream``;
        returns the event that marks them landed.  |desc|^2 and the spatial index
        of the range are computed by whoever consumes them (msfm_stage_plan)."""
        import torch

        a, b = self.row_range(k0, k1)
        if b > a:
            with torch.cuda.stream(copy_stream):
                self.xy[a:b].copy_(self.host.xy[a:b], non_blocking=True)
                self.desc[a:b].copy_(self.host.desc[a:b], non_blocking=True)
        landed = torch.cuda.Event()
        landed.record(copy_stream)
        return landed
    @property
    def h2d_bytes(self) -> int:
        return int(self.xy.numel() * 4 + self.desc.numel() + self.img_off.numel() * 8
                   + self.img_n.numel() * 4 + self.img_wh.numel() * 4)

    def cstruct(self) -> _lib.Bank:
        return _lib.Bank(_lib.ptr(self.xy), _lib.ptr(self.desc), _lib.ptr(self.norm2),
                         _lib.ptr(self.img_off), _lib.ptr(self.img_n), _lib.ptr(self.img_wh),
                         len(self.image_ids), self.n_total)

    def grid(self, D: float, stream=None, build: bool = True) -> "SpatialIndex":
        key = float(D)
        if key not in self._grids:
            self._grids[key] = SpatialIndex(self, key, stream, build=build)
        return self._grids[key]


class SpatialIndex:
    """Subcell ids + row/column bucket CSR tables of every image (msfm_grid_build)."""

    def __init__(self, bank: FeatureBank, D: float, stream=None, build: bool = True):
        import torch

        lib = _lib.load()
        if not D > 0:
            raise ValueError(f"cell half-size d must be positive, got {D}")
        self.D = float(D)
        nimg = len(bank.image_ids)
        dims = np.zeros((nimg, 2), dtype=np.int32)
        buf = (ctypes.c_int32 * 2)()
        for k in range(nimg):
            _lib.check(lib.msfm_grid_dims(int(bank.wh[k, 0]), int(bank.wh[k, 1]), self.D, buf),
                       "msfm_grid_dims")
            dims[k] = (buf[0], buf[1])
        cells = dims[:, 0].astype(np.int64) * dims[:, 1]
        roff = np.zeros(nimg, np.int64)
        if nimg > 1:
            np.cumsum(cells[:-1], out=roff[1:])
        nb = int(cells.sum())
        dev = bank.device
        self.dims = _to_device(dims, dev)
        self.roff = _to_device(roff, dev)
        self.coff = self.roff  # the column table has the same per-image sizes
        self.sub = torch.empty(bank.n_total, dtype=torch.int32, device=dev)
        self.rstart = torch.empty(nb + 1, dtype=torch.int32, device=dev)
        self.cstart = torch.empty(nb + 1, dtype=torch.int32, device=dev)
        self.rmem = torch.empty(max(bank.n_total, 1), dtype=torch.int32, device=dev)
        self.cmem = torch.empty(max(bank.n_total, 1), dtype=torch.int32, device=dev)
        self.rrec = torch.empty((max(bank.n_total, 1), 4), dtype=torch.int32, device=dev)
        self.crec = torch.empty((max(bank.n_total, 1), 4), dtype=torch.int32, device=dev)
        ws_bytes = lib.msfm_grid_workspace_bytes(nb)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        self._bank, self._nb, self._roff_h = bank, nb, roff
        self._ws, self._ws_bytes = ws, ws_bytes
        if not build:
            return
        st = _lib.stream_handle(stream)
        b = bank.cstruct()
        _lib.check(lib.msfm_grid_build(ctypes.byref(b), _lib.ptr(self.dims), _lib.ptr(self.roff),
                                       _lib.ptr(self.coff), nb, bank.n_total, self.D,
                                       _lib.ptr(self.sub), _lib.ptr(self.rstart),
                                       _lib.ptr(self.cstart), _lib.ptr(self.rmem),
                                       _lib.ptr(self.cmem), _lib.ptr(self.rrec),
                                       _lib.ptr(self.crec), _lib.ptr(ws), ws_bytes, st),
                   "msfm_grid_build")

    def bucket_range(self, k0: int, k1: int):
        """Bucket rows [b0, b1) of images [k0, k1) (row and column tables alike)."""
        nimg = len(self._bank.image_ids)
        b0 = int(self._roff_h[k0]) if k0 < nimg else self._nb
        b1 = int(self._roff_h[k1]) if k1 < nimg else self._nb
        return b0, b1

    def build_range(self, k0: int, k1: int, stream=None):
        """Index bank images [k0, k1) only (their rows must be on the device,
        in stream order); ranges built on one stream may come in any order."""
        lib = _lib.load()
        bank = self._bank
        b0, b1 = self.bucket_range(k0, k1)
        f0 = bank.row_range(k0, k1)[0]
        b = bank.cstruct()
        _lib.check(lib.msfm_grid_build_range(ctypes.byref(b), _lib.ptr(self.dims),
                                             _lib.ptr(self.roff), _lib.ptr(self.coff), self._nb,
                                             k0, k1, b0, b1, f0, self.D, _lib.ptr(self.sub),
                                             _lib.ptr(self.rstart), _lib.ptr(self.cstart),
                                             _lib.ptr(self.rmem), _lib.ptr(self.cmem),
                                             _lib.ptr(self.rrec), _lib.ptr(self.crec),
                                             _lib.ptr(self._ws), self._ws_bytes,
                                             _lib.stream_handle(stream)), "msfm_grid_build_range")

    def cstruct(self) -> _lib.Grids:
        return _lib.Grids(_lib.ptr(self.sub), _lib.ptr(self.dims), _lib.ptr(self.roff),
                          _lib.ptr(self.coff), _lib.ptr(self.rstart), _lib.ptr(self.cstart),
                          _lib.ptr(self.rmem), _lib.ptr(self.cmem), _lib.ptr(self.rrec),
                          _lib.ptr(self.crec), self.D)


def _to_device(a: np.ndarray, device):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if device.type == "cuda":
        t = t.pin_memory().to(device, non_blocking=True)
    return t
