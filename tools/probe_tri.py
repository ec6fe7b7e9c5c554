"""Triangulation probe: C4-like long tracks (ring of 489 cameras, tracks of 2-400
views), kernel time of msfm_triangulate_batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1512_06235_b200 import _lib
from paper_1512_06235_b200.triangulation import triangulate_batch

rng = np.random.default_rng(0)
C = 489
ang = np.linspace(0, 2 * np.pi, C, endpoint=False)
K = np.tile(np.array([[2600.0, 0, 1536], [0, 2600.0, 1152], [0, 0, 1]]), (C, 1, 1))
R = np.zeros((C, 3, 3)); t = np.zeros((C, 3))
for c in range(C):
    cen = np.array([8 * np.cos(ang[c]), 0.0, 8 * np.sin(ang[c])])
    z = -cen / np.linalg.norm(cen); x = np.cross([0, 1.0, 0], z); x /= np.linalg.norm(x); y = np.cross(z, x)
    R[c] = np.stack([x, y, z]); t[c] = -R[c] @ cen
T = 21000
lens = np.minimum(2 + rng.geometric(0.02, size=T), 400)
ptr = np.zeros(T + 1, np.int64); np.cumsum(lens, out=ptr[1:])
X = rng.normal(size=(T, 3))
cam = np.empty(ptr[-1], np.int32); pix = np.empty((ptr[-1], 2))
for k in range(T):
    c0 = rng.integers(C)
    cs = (c0 + np.arange(lens[k]) * 2) % C        # a run of neighbouring cameras
    cam[ptr[k]:ptr[k + 1]] = cs
    xc = np.einsum("cij,j->ci", R[cs], X[k]) + t[cs]
    uv = np.einsum("cij,cj->ci", K[cs], xc)
    pix[ptr[k]:ptr[k + 1]] = uv[:, :2] / uv[:, 2:3] + rng.normal(size=(lens[k], 2)) * 0.3
for _ in range(2):
    triangulate_batch(K, R, t, ptr, cam, pix)
torch.cuda.synchronize()
_lib.profile_enable(True)
t0 = time.perf_counter()
st, Xo, err = triangulate_batch(K, R, t, ptr, cam, pix)
dt = time.perf_counter() - t0
ms, n = _lib.profile_read("tri_kernel")
_lib.profile_enable(False)
print(f"tracks {T}, views {ptr[-1]} (mean {lens.mean():.1f}, max {lens.max()}): kernel {ms:.2f} ms, "
      f"call {dt * 1e3:.1f} ms, ok {int((st == 1).sum())}")
