"""Multi-GPU plumbing: one process per GPU, torch.distributed.

Pairs (and query images) are independent given the read-only snapshot, so they
shard with no data-path collective; the only exchange is the final gather of
variable-length match arrays to rank 0, restored to the reference's pair order
(densify.py:238-240).  Works on NCCL (CUDA tensors) and gloo (CPU tensors).
"""

from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int, cost=None) -> np.ndarray:
    """Item indices of this rank.  Without costs: round-robin (pairs sorted by
    image id interleave target images across ranks).  With costs: greedy LPT
    over items sorted by decreasing cost, ties by index (deterministic)."""
    if world <= 1:
        return np.arange(n_items)
    if cost is None:
        return np.arange(rank, n_items, world)
    cost = np.asarray(cost, dtype=np.float64)
    order = np.lexsort((np.arange(n_items), -cost))
    load = np.zeros(world)
    owner = np.empty(n_items, np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += cost[i]
    return np.flatnonzero(owner == rank)


def gather_rows(rows, world: int, dst: int = 0):
    """Variable-length gather of an (n, k) int64 tensor to every rank (all_gather
    of sizes, then of max-padded blocks).  Returns the concatenation on all ranks
    (rank order)."""
    import torch
    import torch.distributed as dist

    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=rows.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(max(sizes), 1)
    buf = torch.zeros((mx, rows.shape[1]), dtype=rows.dtype, device=rows.device)
    buf[:rows.shape[0]] = rows
    out = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return torch.cat([o[:s] for o, s in zip(out, sizes)], 0)


def pack_matches(pair_index, q, t, dist_, ratio):
    """(n, 5) int64 rows: global pair, query fid, target fid, f32 bits of dist/ratio."""
    import torch

    f32 = lambda x: torch.as_tensor(np.asarray(x, np.float32)).view(torch.int32).to(torch.int64)
    return torch.stack([torch.as_tensor(np.asarray(pair_index, np.int64)),
                        torch.as_tensor(np.asarray(q, np.int64)),
                        torch.as_tensor(np.asarray(t, np.int64)), f32(dist_), f32(ratio)], 1)


def unpack_matches(rows):
    """Rows in the reference order (pair, then query id) -> numpy columns."""
    import torch

    r = rows.cpu()
    order = np.lexsort((r[:, 1].numpy(), r[:, 0].numpy()))
    r = r[torch.from_numpy(order)]
    to_f32 = lambda c: c.to(torch.int32).view(torch.float32).numpy()
    return (r[:, 0].numpy(), r[:, 1].numpy().astype(np.int32), r[:, 2].numpy().astype(np.int32),
            to_f32(r[:, 3]), to_f32(r[:, 4]))
