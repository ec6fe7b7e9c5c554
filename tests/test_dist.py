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
