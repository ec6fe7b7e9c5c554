"""GPU parity of the geometry-aware matcher (through the C-ABI) against the
reference's golden outputs and the CPU oracle.  Bit-exact: match index sets,
f32 distances, f32 ratios and SearchStats."""

import numpy as np
import pytest

from golden_io import GUIDED_FIXTURES, STRATEGY_FIXTURES, load

pytestmark = pytest.mark.gpu


def _bank(feature_sets):
    from paper_1512_06235_b200.bank import FeatureBank
    return FeatureBank(feature_sets)


def _assert_same(pair, q, t, d, r):
    np.testing.assert_array_equal(q, pair["mq"])
    np.testing.assert_array_equal(t, pair["mt"])
    np.testing.assert_array_equal(d.astype(np.float64), pair["dist"])
    np.testing.assert_array_equal(r.astype(np.float64), pair["ratio"])


@pytest.mark.parametrize("name", GUIDED_FIXTURES)
def test_batched_matcher_equals_reference_golden(name):
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import match_pairs

    _, scene, _, pairs = load(name)
    bank = _bank(scene.feature_sets)
    F = np.stack([fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]]).F
                  for p in pairs])
    ql = [np.arange(len(scene.feature_sets[p["q"]]), dtype=np.int32) if p["qi"] is None
          else p["qi"] for p in pairs]
    res = match_pairs(bank, [p["q"] for p in pairs], [p["t"] for p in pairs], F, ql,
                      with_stats=True)
    pk, q, t, d, r = res.to_host()
    stats = res.stats.cpu().numpy()
    for k, p in enumerate(pairs):
        sel = pk == k
        _assert_same(p, q[sel], t[sel], d[sel], r[sel])
        np.testing.assert_array_equal(stats[k], p["stats"])


@pytest.mark.parametrize("chunk", [1, 3, 0])
def test_chunking_is_invisible(chunk):
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import match_pairs

    _, scene, _, pairs = load("guided_C1.npz")
    bank = _bank(scene.feature_sets)
    F = np.stack([fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]]).F
                  for p in pairs])
    res = match_pairs(bank, [p["q"] for p in pairs], [p["t"] for p in pairs], F,
                      [p["qi"] for p in pairs], chunk_pairs=chunk)
    pk, q, t, d, r = res.to_host()
    for k, p in enumerate(pairs):
        sel = pk == k
        _assert_same(p, q[sel], t[sel], d[sel], r[sel])


def test_dropin_signature_and_stats():
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import guided_match_pair
    from paper_1512_06235_b200.types import SearchStats

    _, scene, _, pairs = load("guided_unit_s11.npz")
    p = pairs[0]
    geom = fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]])
    st = SearchStats()
    got = guided_match_pair(scene.feature_sets[p["q"]], scene.feature_sets[p["t"]], geom, stats=st)
    q = np.array([m.query.feature_id for m in got])
    t = np.array([m.target.feature_id for m in got])
    d = np.array([m.distance for m in got])
    r = np.array([m.ratio for m in got])
    _assert_same(p, q, t, d, r)
    assert (st.queries, st.candidates) == tuple(p["stats"])
    assert all(m.query.image_id == p["q"] and m.target.image_id == p["t"] for m in got)


def test_dropin_edge_cases():
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import guided_match_pair

    _, scene, _, pairs = load("guided_unit_s12.npz")
    fq, ft = scene.feature_sets[0], scene.feature_sets[1]
    geom = fundamental_from_poses(scene.cameras[0], scene.cameras[1])
    assert guided_match_pair(fq, ft, geom, target_indices=np.array([], dtype=int)) == []
    assert guided_match_pair(fq, ft, geom, query_indices=np.array([], dtype=int)) == []
    with pytest.raises(ValueError):
        guided_match_pair(fq, ft, geom, strategy="bogus")
    with pytest.raises(ValueError):
        guided_match_pair(fq, ft, geom, d=0.0)


def test_degenerate_pair_is_skipped():
    from paper_1512_06235_b200.guided import match_pairs

    _, scene, _, pairs = load("guided_unit_s9.npz")
    bank = _bank(scene.feature_sets)
    F = np.full((1, 3, 3), np.nan)
    res = match_pairs(bank, [0], [1], F, [np.arange(len(scene.feature_sets[0]), dtype=np.int32)])
    assert int(res.count.cpu()[0]) == 0


@pytest.mark.parametrize("n_cams,seed_pairs", [(14, 0)])
def test_8k_scene_matches_oracle(n_cams, seed_pairs):
    """C2/C3 feature density (8k/img, 3072x2304): every densify pair of a
    14-camera scene, batched, against the C oracle."""
    from oracle import guided as og
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import match_pairs

    scene, snap = scenes.build("C3", n_cameras=n_cams)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, with_stats=True)
    pk, q, t, d, r = res.to_host()
    stats = res.stats.cpu().numpy()
    total = 0
    for j, k in enumerate(ok):
        fq, ft = scene.feature_sets[int(wl.q_img[k])], scene.feature_sets[int(wl.t_img[k])]
        oq, ot, od, orr, ost = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                               ft.width, ft.height, wl.F[k], ql[j])
        sel = pk == j
        np.testing.assert_array_equal(q[sel], oq)
        np.testing.assert_array_equal(t[sel], ot)
        np.testing.assert_array_equal(d[sel], od)
        np.testing.assert_array_equal(r[sel], orr)
        np.testing.assert_array_equal(stats[j], ost)
        total += len(oq)
    assert total > 1000


def test_shared_query_lists_and_packed_rows():
    """Pairs that pass one list object share its upload (d_qlist_src); the
    result, packed on the device into 16-B rows, must not depend on it."""
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import MATCH_ROW, match_pairs

    scene, snap = scenes.build("C1", n_cameras=10)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(scene.feature_sets)
    shared = [wl.untracked[int(wl.q_img[k])] for k in ok]
    copied = [np.array(x, copy=True) for x in shared]
    a = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], shared, chunk_pairs=3)
    b = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], copied)
    ra, rb = a.rows_host(), b.rows_host()
    assert ra.dtype == MATCH_ROW and len(ra) > 100
    np.testing.assert_array_equal(ra.view(np.int32), rb.view(np.int32))
    pk, q, t, d, r = b.to_host()
    np.testing.assert_array_equal(pk, ra["pair"])
    np.testing.assert_array_equal(q, ra["q"])
    np.testing.assert_array_equal(t, ra["t"])
    np.testing.assert_array_equal(d, ra["dist"])
    assert np.all(np.diff(pk) >= 0)
    cnt = b.count.cpu().numpy()
    np.testing.assert_array_equal(np.bincount(pk, minlength=len(ok)), cnt)


@pytest.mark.parametrize("name", STRATEGY_FIXTURES)
def test_linear_and_radial_strategies_equal_reference(name):
    """strategy="linear" (rep-line band, guided.py:190-194) and "radial" (disks of
    radius d*sqrt(2) around the samples, guided.py:273-285): match sets and
    SearchStats identical to the reference's."""
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import match_pairs

    strategy = name.split("_")[1]
    _, scene, _, pairs = load(name)
    bank = _bank(scene.feature_sets)
    F = np.stack([fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]]).F
                  for p in pairs])
    ql = [np.arange(len(scene.feature_sets[p["q"]]), dtype=np.int32) if p["qi"] is None
          else p["qi"] for p in pairs]
    res = match_pairs(bank, [p["q"] for p in pairs], [p["t"] for p in pairs], F, ql,
                      with_stats=True, strategy=strategy)
    pk, q, t, d, r = res.to_host()
    stats = res.stats.cpu().numpy()
    for k, p in enumerate(pairs):
        sel = pk == k
        _assert_same(p, q[sel], t[sel], d[sel], r[sel])
        np.testing.assert_array_equal(stats[k], p["stats"])
    # and without stats (super-group path)
    res = match_pairs(bank, [p["q"] for p in pairs], [p["t"] for p in pairs], F, ql,
                      strategy=strategy)
    pk, q, t, d, r = res.to_host()
    for k, p in enumerate(pairs):
        sel = pk == k
        _assert_same(p, q[sel], t[sel], d[sel], r[sel])


def test_dropin_strategies_and_errors():
    from paper_1512_06235_b200.geometry import fundamental_from_poses
    from paper_1512_06235_b200.guided import guided_match_pair
    from paper_1512_06235_b200.types import SearchStats

    _, scene, _, pairs = load("strategy_radial_s9.npz")
    p = pairs[0]
    geom = fundamental_from_poses(scene.cameras[p["q"]], scene.cameras[p["t"]])
    st = SearchStats()
    ms = guided_match_pair(scene.feature_sets[p["q"]], scene.feature_sets[p["t"]], geom,
                           strategy="radial", stats=st)
    np.testing.assert_array_equal([m.query.feature_id for m in ms], p["mq"])
    assert (st.queries, st.candidates) == tuple(p["stats"])
    with pytest.raises(ValueError):
        guided_match_pair(scene.feature_sets[p["q"]], scene.feature_sets[p["t"]], geom,
                          strategy="bogus")


@pytest.mark.parametrize("chunk", [1, 3, 0])
def test_pipelined_host_rows_equal_device_packing(chunk):
    """msfm_guided_match_rows (chunk-pipelined pack + D2H) == match_pairs + packing."""
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import match_pairs, match_pairs_rows

    scene, snap = scenes.build("C1", n_cameras=10)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    want = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql).rows_host()
    got = match_pairs_rows(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, chunk_pairs=chunk)
    assert len(got) == len(want) > 100
    np.testing.assert_array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("seg,chunk,first", [(1, 7, 0), (3, 16, 5), (2, 0, 3), (64, 0, 128)])
def test_staged_upload_rows_equal_resident_bank(seg, chunk, first):
    """match_pairs_rows_staged (bank uploaded and indexed range by range while the
    chunks match) == match_pairs_rows over a fully resident bank."""
    import torch

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import HostBank
    from paper_1512_06235_b200.guided import match_pairs_rows, match_pairs_rows_staged

    scene, snap = scenes.build("C1", n_cameras=10)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    want = match_pairs_rows(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, chunk_pairs=chunk)
    host = HostBank(scene.feature_sets)
    got, b2 = match_pairs_rows_staged(host, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql,
                                      segment_images=seg, chunk_pairs=chunk,
                                      first_chunk_pairs=first)
    torch.cuda.synchronize()
    assert len(got) == len(want) > 100
    np.testing.assert_array_equal(got.view(np.int32), want.view(np.int32))
    # the staged bank ends complete: rows, norms, CSR starts identical
    assert torch.equal(b2.desc, bank.desc) and torch.equal(b2.norm2, bank.norm2)
    g1, g2 = bank.grid(10.0), b2.grid(10.0)        # D = d * inflation = 8 * 1.25
    for name in ("sub", "rstart", "cstart"):
        assert torch.equal(getattr(g1, name), getattr(g2, name)), name


def test_grid_build_ranges_any_order_equal_full_build():
    """msfm_grid_build_range over shuffled image ranges == msfm_grid_build (bucket
    members compared as sets: the scatter order inside a bucket is atomic)."""
    import torch

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import SpatialIndex

    scene, _ = scenes.build("C1", n_cameras=9)
    bank = _bank(scene.feature_sets)
    full = bank.grid(10.0)
    part = SpatialIndex(bank, 10.0, build=False)
    cuts = [0, 1, 4, 5, 9]
    for k in [2, 0, 3, 1]:
        part.build_range(cuts[k], cuts[k + 1])
    torch.cuda.synchronize()
    for name in ("sub", "rstart", "cstart"):
        assert torch.equal(getattr(full, name), getattr(part, name)), name
    rs = full.rstart.cpu().numpy()
    for mem in ("rmem", "cmem"):
        a, b = getattr(full, mem).cpu().numpy(), getattr(part, mem).cpu().numpy()
        st = rs if mem == "rmem" else full.cstart.cpu().numpy()
        key = np.repeat(np.arange(len(st) - 1), np.diff(st))
        assert np.array_equal(np.sort(a + key.astype(np.int64) * 100000),
                              np.sort(b + key.astype(np.int64) * 100000))


def test_16k_feature_pairs_match_oracle():
    """C4/C5 feature density (16k/img): a few densify pairs against the C oracle
    (16-bit feature ids in the packed rows, larger strips and member sets)."""
    from oracle import guided as og
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import match_pairs

    spec = scenes.spec_for("C4", n_cameras=12)
    scene = scenes.generate_scene(spec)
    snap = scenes.coarse_snapshot(scene, range(12))
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)[:3]
    bank = _bank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    res = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql, with_stats=True)
    pk, q, t, d, r = res.to_host()
    stats = res.stats.cpu().numpy()
    assert max(len(scene.feature_sets[i]) for i in scene.feature_sets) > 15000
    for j, k in enumerate(ok):
        fq, ft = scene.feature_sets[int(wl.q_img[k])], scene.feature_sets[int(wl.t_img[k])]
        oq, ot, od, orr, ost = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                               ft.width, ft.height, wl.F[k], ql[j])
        sel = pk == j
        np.testing.assert_array_equal(q[sel], oq)
        np.testing.assert_array_equal(t[sel], ot)
        np.testing.assert_array_equal(d[sel], od)
        np.testing.assert_array_equal(r[sel], orr)
        np.testing.assert_array_equal(stats[j], ost)


def test_bench_workload_sample_matches_oracle():
    """The bench's own C3 step (all 5,401 pairs of the 320-camera scene in one call):
    a seeded sample of pairs equals the C oracle (tools/parity_sweep.py does 256)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import guided as og
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import match_pairs

    scene, snap = scenes.build("C3", n_cameras=320)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(scene.feature_sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    pk, q, t, d, r = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql).to_host()
    pick = np.random.default_rng(7).choice(len(ok), size=48, replace=False)

    def one(j):
        k = int(ok[j])
        qi, ti = int(wl.q_img[k]), int(wl.t_img[k])
        fq, ft = scene.feature_sets[qi], scene.feature_sets[ti]
        oq, ot, od, orr, _ = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                             ft.width, ft.height, wl.F[k], wl.untracked[qi])
        sel = pk == j
        return (np.array_equal(q[sel], oq) and np.array_equal(t[sel], ot)
                and np.array_equal(d[sel], od) and np.array_equal(r[sel], orr))

    with ThreadPoolExecutor(8) as ex:
        assert all(ex.map(one, pick))


def test_staged_rows_with_empty_lists_and_images():
    """match_pairs_rows_staged with empty query lists, a zero-feature image and a
    degenerate (NaN) F: identical to the resident path."""
    import torch

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import HostBank
    from paper_1512_06235_b200.guided import match_pairs_rows, match_pairs_rows_staged
    from paper_1512_06235_b200.types import FeatureSet

    scene, snap = scenes.build("C1", n_cameras=8)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    sets = dict(scene.feature_sets)
    empty_id = max(sets) + 1
    sets[empty_id] = FeatureSet(image_id=empty_id, width=640, height=480,
                                xy=np.zeros((0, 2), np.float32), scale=np.zeros(0, np.float32),
                                orientation=np.zeros(0, np.float32),
                                descriptors=np.zeros((0, 128), np.uint8))
    q = list(wl.q_img[ok]) + [int(wl.q_img[ok[0]]), empty_id]
    t = list(wl.t_img[ok]) + [empty_id, int(wl.t_img[ok[0]])]
    F = np.concatenate([wl.F[ok], np.full((1, 3, 3), np.nan), wl.F[ok[:1]]])
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    ql[1] = np.zeros(0, np.int32)                          # a pair with no queries
    ql += [wl.untracked[int(wl.q_img[ok[0]])], np.zeros(0, np.int32)]
    bank = _bank(sets)
    want = match_pairs_rows(bank, q, t, F, ql, chunk_pairs=5)
    got, _ = match_pairs_rows_staged(HostBank(sets), q, t, F, ql, chunk_pairs=5,
                                     segment_images=2, first_chunk_pairs=3)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.view(np.int32), want.view(np.int32))


@pytest.mark.parametrize("ratio", [1.5, 4.0])
def test_ratio_above_one_ties_resolve_to_lowest_target(ratio):
    """ratio > 1 (the reference accepts any ratio, matching.py:82-103): a tie at the
    minimum distance is then accepted with ratio 1 and names the lowest target id
    among the tied candidates (np.argmin over the sorted candidate list,
    guided.py:460).  Ties are forced by copying each target feature's descriptor onto
    its nearest neighbour in the image; every pair of a small C3 scene against the C
    oracle, bit-exact."""
    import dataclasses

    from oracle import guided as og
    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.guided import match_pairs

    scene, snap = scenes.build("C3", n_cameras=6)
    rng = np.random.default_rng(7)
    sets = {}
    for i, fs in scene.feature_sets.items():
        desc = np.array(fs.descriptors, copy=True)
        xy = np.asarray(fs.xy, np.float64)
        pick = rng.choice(len(desc), size=len(desc) // 3, replace=False)
        for j in pick:       # nearest other feature takes j's descriptor
            d2 = ((xy - xy[j]) ** 2).sum(axis=1)
            d2[j] = np.inf
            desc[int(np.argmin(d2))] = desc[j]
        sets[i] = dataclasses.replace(fs, descriptors=desc)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    bank = _bank(sets)
    ql = [wl.untracked[int(wl.q_img[k])] for k in ok]
    pk, q, t, d, r = match_pairs(bank, wl.q_img[ok], wl.t_img[ok], wl.F[ok], ql,
                                 ratio=ratio).to_host()
    ties = total = 0
    for j, k in enumerate(ok):
        fq, ft = sets[int(wl.q_img[k])], sets[int(wl.t_img[k])]
        oq, ot, od, orr, _ = og.guided_match(fq.xy, fq.descriptors, ft.xy, ft.descriptors,
                                             ft.width, ft.height, wl.F[k], ql[j], ratio=ratio)
        sel = pk == j
        np.testing.assert_array_equal(q[sel], oq)
        np.testing.assert_array_equal(t[sel], ot)
        np.testing.assert_array_equal(d[sel], od)
        np.testing.assert_array_equal(r[sel], orr)
        ties += int((orr == 1.0).sum())
        total += len(oq)
    assert total > 1000 and ties > 50, (total, ties)
