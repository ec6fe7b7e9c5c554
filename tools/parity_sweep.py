"""Parity at the benchmark's own sizes (not a benchmark): the device results of
the bench workloads against the CPU oracle on seeded samples.

  * C3 (bench matcher workload, 320 cameras, 8k features): every pair matched on
    the device in one call; a seeded sample of pairs re-run by the C oracle
    (oracle/guided_oracle.c) — match sets, f32 distances and ratios identical.
  * C4 (16k features): the same on a sample of its densify pairs.
  * C2 (bench localization workload, 80 query images): direct 3D-2D search on the
    device vs the exact oracle for every image, and the seeded PnP-RANSAC inlier
    masks vs the oracle's for every image that reaches PnP.

    python tools/parity_sweep.py [n_sample=256]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from oracle import guided as og
from oracle import localize as ol
from paper_1512_06235_b200 import scenes
from paper_1512_06235_b200.bank import FeatureBank
from paper_1512_06235_b200.guided import match_pairs
from paper_1512_06235_b200.localize import PointSet, direct_search
from paper_1512_06235_b200.pnp import pnp_batch

n_sample = int(sys.argv[1]) if len(sys.argv) > 1 else 256
og.lib()


def matcher_sweep(config, n_cameras, n_pick, seed):
    t0 = time.perf_counter()
    # every camera registered (the densify pair set over all of them)
    scene = scenes.generate_scene(scenes.spec_for(config, n_cameras))
    snap = scenes.coarse_snapshot(scene, list(range(n_cameras)))
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = FeatureBank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql)
    pk, q, t, d, r = res.to_host()
    pick = np.random.default_rng(seed).choice(len(ok), size=min(n_pick, len(ok)), replace=False)

    def one(j):
        k = int(ok[j])
        qi, ti = int(wl.q_img[k]), int(wl.t_img[k])
        fq, ft = scene.feature_sets[qi], scene.feature_sets[ti]
        oq, ot, od, orr, _ = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                             ft.width, ft.height, wl.F[k], wl.untracked[qi])
        sel = pk == j
        same = (np.array_equal(q[sel], oq) and np.array_equal(t[sel], ot)
                and np.array_equal(d[sel], od) and np.array_equal(r[sel], orr))
        return same, len(oq)

    with ThreadPoolExecutor(os.cpu_count()) as ex:
        out = list(ex.map(one, pick))
    bad = sum(1 for s, _ in out if not s)
    print(f"{config}: {len(ok)} pairs matched on the device ({int(len(pk))} matches); "
          f"{len(pick)} seeded pairs vs the C oracle: {len(pick) - bad} identical, {bad} differ "
          f"({sum(n for _, n in out)} matches compared; {time.perf_counter() - t0:.0f} s)",
          flush=True)
    return bad


def localization_sweep():
    t0 = time.perf_counter()
    scene, snap, queries = bench.build_localization()
    S, n = scenes.track_sums(scene, snap)
    pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
    bank = FeatureBank({q: scene.feature_sets[q] for q in queries})
    corrs = direct_search(bank, pts, queries)
    bad_corr = 0
    for s, qimg in enumerate(queries):
        want = ol.direct_3d2d(np.arange(len(S)), S, n, scene.feature_sets[qimg].descriptors)
        bad_corr += not np.array_equal(corrs[s], want)
    todo = [k for k, c in enumerate(corrs) if len(c) > 16]
    X = [snap.point_xyz[corrs[k][:, 0]] for k in todo]
    uv = [scene.feature_sets[queries[k]].xy[corrs[k][:, 1]].astype(np.float64) for k in todo]
    Ks = [scene.cameras[queries[k]].K for k in todo]
    res = pnp_batch(X, uv, Ks, [queries[k] for k in todo])
    bad_pnp, rot = 0, []
    for j, k in enumerate(todo):
        try:
            o = ol.pnp_ransac(X[j], uv[j], Ks[j], seed=queries[k])
            ost = "ok" if o is not None else "none"
        except OverflowError:
            o, ost = None, "overflow"
        r = res[j]
        if r.status != ost:
            bad_pnp += 1
            continue
        if ost == "ok":
            if not np.array_equal(r.mask, o[2]):
                bad_pnp += 1
            rot.append(float(np.abs(r.R - o[0]).max()))
    print(f"C2: {len(queries)} images, direct 3D-2D correspondences identical for "
          f"{len(queries) - bad_corr}; PnP-RANSAC status + inlier mask identical for "
          f"{len(todo) - bad_pnp} of {len(todo)} (max |R - R_oracle| "
          f"{max(rot) if rot else 0:.1e}; {time.perf_counter() - t0:.0f} s)", flush=True)
    return bad_corr + bad_pnp


bad = matcher_sweep("C3", 320, n_sample, 0)
bad += localization_sweep()
bad += matcher_sweep("C4", 160, max(n_sample // 4, 16), 1)
print("PARITY SWEEP:", "all identical" if bad == 0 else f"{bad} differences", flush=True)
