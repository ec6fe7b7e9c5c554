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


def chunk_bounds(n_items: int, n_chunks: int) -> np.ndarray:
    """Contiguous split of n_items into n_chunks nearly equal chunks (bounds array)."""
    n_chunks = max(1, min(n_chunks, max(n_items, 1)))
    return np.linspace(0, n_items, n_chunks + 1).round().astype(np.int64)


class ChunkGather:
    """Gather to rank 0, chunk by chunk, of packed 16-B match rows.

    Every rank knows every rank's chunk capacities (``caps[r][k]``: the chunk's query
    count — a query yields at most one row), so buffers are sized without a count
    exchange: rank r sends chunk k's capacity-sized row buffer and its row count as
    soon as the chunk is packed (NCCL runs after the chunk's kernels on its own
    stream, overlapping chunk k+1's matching); rank 0 posts the matching receives on
    a side stream so they never wait on its own compute.  On gloo (CPU tests) the
    same protocol runs on host tensors.  Rank 0's ``finish()`` returns
    {(rank, chunk): (rows (cap, 4) int32, count (1,) int64)}; other ranks get None."""

    def __init__(self, world: int, rank: int, caps, device=None):
        import torch
        import torch.distributed as dist

        self.world, self.rank, self.caps = world, rank, caps
        self.gloo = dist.get_backend() == "gloo"
        self.dev = torch.device("cpu") if self.gloo else device
        self.side = None if (self.gloo or device is None) else torch.cuda.Stream(device)
        self.works, self.keep, self.got = [], [], {}

    def put(self, k: int, rows, count):
        import torch
        import torch.distributed as dist

        if self.rank != 0:
            cap = int(self.caps[self.rank][k])
            r = rows[:max(cap, 1)].contiguous()
            c = count.reshape(1).to(torch.int64)
            if self.gloo:
                r, c = r.cpu(), c.cpu()
            self.keep += [r, c]
            self.works += [dist.isend(r, 0), dist.isend(c, 0)]
            return
        self.got[(0, k)] = (rows, count)
        for src in range(1, self.world):
            buf = torch.empty((max(int(self.caps[src][k]), 1), 4), dtype=torch.int32, device=self.dev)
            cnt = torch.empty(1, dtype=torch.int64, device=self.dev)
            if self.side is not None:
                with torch.cuda.stream(self.side):
                    self.works += [dist.irecv(buf, src), dist.irecv(cnt, src)]
            else:
                self.works += [dist.irecv(buf, src), dist.irecv(cnt, src)]
            self.got[(src, k)] = (buf, cnt)

    def finish(self):
        for w in self.works:
            w.wait()
        self.works, self.keep = [], []
        return self.got if self.rank == 0 else None


def merge_chunk_rows(got, pair_index):
    """Rank 0: the gathered chunks as one host MATCH_ROW-like int32 (n, 4) array in
    the reference's pair order.  ``pair_index[(rank, chunk)]`` maps a chunk's local
    pair index to the global one."""
    out = []
    for key in sorted(got):
        rows, cnt = got[key]
        n = int(cnt.reshape(-1)[0].item())
        r = rows[:n].cpu().numpy().copy()
        r[:, 0] = np.asarray(pair_index[key], np.int64)[r[:, 0]]
        out.append(r)
    if not out:
        return np.zeros((0, 4), np.int32)
    allr = np.concatenate(out)
    order = np.lexsort(((allr[:, 1] & 0xFFFF), allr[:, 0]))
    return allr[order]


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
