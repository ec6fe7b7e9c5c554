"""Multi-rank host logic on CPU (gloo, world_size 2): sharding covers every item
once and the gathered matches equal the single-process result in pair order."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1512_06235_b200.dist import shard


def test_shard_partitions():
    for world in (1, 2, 3, 8):
        got = np.sort(np.concatenate([shard(101, r, world) for r in range(world)]))
        np.testing.assert_array_equal(got, np.arange(101))
    cost = np.random.default_rng(0).uniform(1, 10, 57)
    parts = [shard(57, r, 4, cost) for r in range(4)]
    np.testing.assert_array_equal(np.sort(np.concatenate(parts)), np.arange(57))
    loads = [cost[p].sum() for p in parts]
    assert max(loads) - min(loads) <= cost.max()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_pairs, out_path):
    import torch.distributed as dist

    from paper_1512_06235_b200.dist import gather_rows, pack_matches, unpack_matches

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(123)
    # deterministic fake per-pair matches (what each pair's matcher would emit)
    per_pair = []
    for k in range(n_pairs):
        m = int(rng.integers(0, 7))
        q = np.sort(rng.choice(1000, m, replace=False))
        per_pair.append((q, rng.integers(0, 900, m), rng.random(m), rng.random(m)))
    mine = shard(n_pairs, rank, world)
    pk = np.concatenate([[k] * len(per_pair[k][0]) for k in mine]) if len(mine) else np.zeros(0)
    cols = [np.concatenate([per_pair[k][c] for k in mine]) for c in range(4)]
    rows = pack_matches(pk, *cols)
    allrows = gather_rows(rows, world)
    if rank == 0:
        np.save(out_path, np.stack([np.asarray(c, np.float64) for c in unpack_matches(allrows)]))
    dist.destroy_process_group()


def test_gloo_gather_restores_pair_order(tmp_path):
    world, n_pairs = 2, 37
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(world, _free_port(), n_pairs, out), nprocs=world, join=True)
    got = np.load(out)
    rng = np.random.default_rng(123)
    ref = [[], [], [], [], []]
    for k in range(n_pairs):
        m = int(rng.integers(0, 7))
        q = np.sort(rng.choice(1000, m, replace=False))
        t, d, r = rng.integers(0, 900, m), rng.random(m), rng.random(m)
        ref[0] += [k] * m; ref[1] += list(q); ref[2] += list(t)
        ref[3] += list(np.float32(d)); ref[4] += list(np.float32(r))
    np.testing.assert_array_equal(got, np.array(ref, np.float64))


def _merge_gather_worker(rank, world, port, n_pairs, out_path):
    """bench.track_merge_leg's N > 1 gather: each rank's rows carry rank-local pair
    indices (its call over ok[rank::world]); mapped to rank + world * local they
    index the global pair list on rank 0."""
    import torch
    import torch.distributed as dist

    from paper_1512_06235_b200.dist import gather_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(n_pairs, rank, world)
    # one row per match; pair j of this rank has (global pair % 5) matches
    rows = []
    for j, k in enumerate(mine):
        for m in range(int(k) % 5):
            rows.append([j, int(k) * 10 + m, 0, 0])
    rows = torch.tensor(rows if rows else np.zeros((0, 4)), dtype=torch.int32).reshape(-1, 4)
    g = rows.clone()
    g[:, 0] = rank + world * g[:, 0]
    allrows = gather_rows(g, world)
    if rank == 0:
        np.save(out_path, allrows.numpy())
    dist.destroy_process_group()


def test_gloo_merge_gather_maps_local_pairs_to_global():
    world, n_pairs = 2, 23
    out = os.path.join(os.environ.get("TMPDIR", "/tmp"), f"mg_{os.getpid()}.npy")
    mp.spawn(_merge_gather_worker, args=(world, _free_port(), n_pairs, out), nprocs=world,
             join=True)
    got = np.load(out)
    os.remove(out)
    # every match's global pair index agrees with the payload written for that pair
    np.testing.assert_array_equal(got[:, 1] // 10, got[:, 0])
    want = sorted((k, k * 10 + m) for k in range(n_pairs) for m in range(k % 5))
    assert sorted(map(tuple, got[:, :2].tolist())) == want


def _chunk_worker(rank, world, port, n_pairs, n_chunks, out_path):
    """bench's N > 1 data plane on CPU: each rank's pairs in chunks, every chunk's
    capacity-sized row buffer + count to rank 0 (ChunkGather), merged in pair order."""
    import torch
    import torch.distributed as dist

    from paper_1512_06235_b200.dist import ChunkGather, chunk_bounds, merge_chunk_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nq = np.arange(n_pairs) % 7 + 1                  # queries per pair (capacity)
    caps, index = [], {}
    for r in range(world):
        mr = np.arange(r, n_pairs, world)
        b = chunk_bounds(len(mr), n_chunks)
        caps.append([int(nq[mr[b[k]:b[k + 1]]].sum()) for k in range(len(b) - 1)])
        for k in range(len(b) - 1):
            index[(r, k)] = mr[b[k]:b[k + 1]]
    mine = np.arange(rank, n_pairs, world)
    b = chunk_bounds(len(mine), n_chunks)
    gat = ChunkGather(world, rank, caps)
    for k in range(len(b) - 1):
        rows = []
        for j, p in enumerate(mine[b[k]:b[k + 1]]):
            for q in range(int(p) % 3):                 # p % 3 matches per pair, q < nq
                rows.append([j, q | ((int(p) * 10 + q) << 16), int(p), q])
        cap = max(caps[rank][k], 1)
        buf = torch.full((cap, 4), -7, dtype=torch.int32)
        if rows:
            buf[:len(rows)] = torch.tensor(rows, dtype=torch.int32)
        gat.put(k, buf, torch.tensor([len(rows)], dtype=torch.int64))
    got = gat.finish()
    if rank == 0:
        np.save(out_path, merge_chunk_rows(got, index))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_chunks", [1, 3])
def test_gloo_chunk_gather_to_rank0(tmp_path, n_chunks):
    world, n_pairs = 2, 29
    out = str(tmp_path / "c.npy")
    mp.spawn(_chunk_worker, args=(world, _free_port(), n_pairs, n_chunks, out), nprocs=world,
             join=True)
    got = np.load(out)
    want = np.array([[p, q | ((p * 10 + q) << 16), p, q] for p in range(n_pairs)
                     for q in range(p % 3)], np.int32)
    np.testing.assert_array_equal(got, want)


def _gpu_worker(rank, world, port, out_path):
    """Two ranks on cuda:0 (gloo for the host collectives): the real matcher over
    each rank's pair shard in chunks, rows gathered to rank 0; the real direct 3D-2D
    search over each rank's image shard, correspondences gathered to rank 0."""
    import torch
    import torch.distributed as dist

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.dist import ChunkGather, chunk_bounds, merge_chunk_rows
    from paper_1512_06235_b200.guided import match_pairs
    from paper_1512_06235_b200.localize import PointSet, direct_search

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    scene, snap = scenes.build("C1", n_cameras=14)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    qn = np.array([len(wl.untracked[int(wl.q_img[k])]) for k in ok], np.int64)
    caps, index = [], {}
    for r in range(world):
        mr = np.arange(r, len(ok), world)
        b = chunk_bounds(len(mr), 3)
        caps.append([int(qn[mr[b[k]:b[k + 1]]].sum()) for k in range(len(b) - 1)])
        for k in range(len(b) - 1):
            index[(r, k)] = mr[b[k]:b[k + 1]]
    bank = FeatureBank(scene.feature_sets)
    mine = np.arange(rank, len(ok), world)
    b = chunk_bounds(len(mine), 3)
    gat = ChunkGather(world, rank, caps, torch.device("cuda", 0))
    for k in range(len(b) - 1):
        sel = ok[mine[b[k]:b[k + 1]]]
        res = match_pairs(bank, wl.q_img[sel], wl.t_img[sel], wl.F[sel],
                          [wl.untracked[int(wl.q_img[j])] for j in sel])
        rows, cnt = res.packed_device()
        gat.put(k, rows, cnt)
    got = gat.finish()
    # localization: images round-robin
    reg = set(int(i) for i in snap.registered)
    S, n = scenes.track_sums(scene, snap)
    pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
    imgs = sorted(scene.feature_sets)[rank::world]
    corr = direct_search(FeatureBank({i: scene.feature_sets[i] for i in imgs}), pts, imgs)
    parts = [None] * world if rank == 0 else None
    dist.gather_object(list(zip(imgs, [c.tolist() for c in corr])), parts, dst=0)
    if rank == 0:
        merged = merge_chunk_rows(got, index)
        loc = dict(kv for p in parts for kv in p)
        np.save(out_path, merged)
        import pickle
        with open(out_path + ".loc", "wb") as f:
            pickle.dump(loc, f)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_equal_single_process(tmp_path):
    """byte-identical merged rows / correspondences vs one process."""
    import pickle

    from paper_1512_06235_b200 import scenes
    from paper_1512_06235_b200.bank import FeatureBank
    from paper_1512_06235_b200.guided import match_pairs
    from paper_1512_06235_b200.localize import PointSet, direct_search

    out = str(tmp_path / "two.npy")
    mp.spawn(_gpu_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    scene, snap = scenes.build("C1", n_cameras=14)
    wl = scenes.pair_workload(scene, snap)
    ok = np.flatnonzero(wl.valid)
    res = match_pairs(FeatureBank(scene.feature_sets), wl.q_img[ok], wl.t_img[ok], wl.F[ok],
                      [wl.untracked[int(wl.q_img[k])] for k in ok])
    rows, _ = res.packed()
    want = rows.cpu().numpy()
    assert len(want) > 1000
    np.testing.assert_array_equal(got, want)
    with open(out + ".loc", "rb") as f:
        loc = pickle.load(f)
    S, n = scenes.track_sums(scene, snap)
    pts = PointSet(S=S, n=n, ids=np.arange(len(S)))
    imgs = sorted(scene.feature_sets)
    corr = direct_search(FeatureBank(scene.feature_sets), pts, imgs)
    assert sorted(loc) == imgs
    for i, c in zip(imgs, corr):
        assert loc[i] == c.tolist()
