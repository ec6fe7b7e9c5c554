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


class HostBank:
    """Concatenated feature arrays in pinned host memory (the H2D staging area)."""

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

    def __init__(self, feature_sets=None, device=None, image_ids=None, stream=None, host=None):
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
        self.xy = host.xy.to(dev, non_blocking=True)
        self.desc = host.desc.to(dev, non_blocking=True)
        self.img_off = host.img_off.to(dev, non_blocking=True)
        self.img_n = host.img_n.to(dev, non_blocking=True)
        self.img_wh = host.img_wh.to(dev, non_blocking=True)
        self.norm2 = torch.empty(self.n_total, dtype=torch.int32, device=dev)
        st = _lib.stream_handle(stream)
        _lib.check(lib.msfm_feature_norms(_lib.ptr(self.desc), self.n_total,
                                          _lib.ptr(self.norm2), st), "msfm_feature_norms")
        self.max_n = int(self.counts.max()) if len(self.counts) else 0
        self._grids = {}

    @property
    def h2d_bytes(self) -> int:
        return int(self.xy.numel() * 4 + self.desc.numel() + self.img_off.numel() * 8
                   + self.img_n.numel() * 4 + self.img_wh.numel() * 4)

    def cstruct(self) -> _lib.Bank:
        return _lib.Bank(_lib.ptr(self.xy), _lib.ptr(self.desc), _lib.ptr(self.norm2),
                         _lib.ptr(self.img_off), _lib.ptr(self.img_n), _lib.ptr(self.img_wh),
                         len(self.image_ids), self.n_total)

    def grid(self, D: float, stream=None) -> "SpatialIndex":
        key = float(D)
        if key not in self._grids:
            self._grids[key] = SpatialIndex(self, key, stream)
        return self._grids[key]


class SpatialIndex:
    """Subcell ids + row/column bucket CSR tables of every image (msfm_grid_build)."""

    def __init__(self, bank: FeatureBank, D: float, stream=None):
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
        st = _lib.stream_handle(stream)
        b = bank.cstruct()
        _lib.check(lib.msfm_grid_build(ctypes.byref(b), _lib.ptr(self.dims), _lib.ptr(self.roff),
                                       _lib.ptr(self.coff), nb, bank.n_total, self.D,
                                       _lib.ptr(self.sub), _lib.ptr(self.rstart),
                                       _lib.ptr(self.cstart), _lib.ptr(self.rmem),
                                       _lib.ptr(self.cmem), _lib.ptr(self.rrec),
                                       _lib.ptr(self.crec), _lib.ptr(ws), ws_bytes, st),
                   "msfm_grid_build")
        self._ws = ws  # keep alive until the stream has consumed it

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
