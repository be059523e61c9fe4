"""Multi-GPU sharding of the geometry stage.

Batches are independent (SPEC: "batches may be processed concurrently and results concatenated
in batch order"), so the index stream is cut into contiguous ranges of WHOLE batches, one range
per rank, with the vertex buffer replicated.  No collective sits on the data path; the only
exchange is the reduction of the statistics block (SUM for the counters, MAX for the longest
probe chain), which is what the reference's ordered merge does (strategies.py:472-483).
Multi-draw workloads are sharded by whole draws (longest-processing-time bin packing)."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N

SUM_WORDS = (N.VR_STAT_INDICES, N.VR_STAT_INVOCATIONS, N.VR_STAT_BATCHES, N.VR_STAT_ROUNDS,
             N.VR_STAT_PROBES_FAST, N.VR_STAT_PROBES_SLOW)
MAX_WORDS = (N.VR_STAT_PROBE_MAX_CHAIN,)


def shard_range(n_items: int, rank: int, world: int):
    """Balanced contiguous split: the first n % world ranks get one extra item."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_batches(offsets, rank: int, world: int):
    """Offsets array (n_batches+1) -> this rank's sub-array (whole batches, contiguous)."""
    nb = max(len(offsets) - 1, 0)
    lo, hi = shard_range(nb, rank, world)
    return offsets[lo:hi + 1] if hi > lo else offsets[:0]


def lpt_assign(sizes, world: int):
    """Whole draws to ranks, largest first onto the least-loaded rank (ties: lowest rank).
    Returns a list of index arrays, each in ascending draw order."""
    sizes = np.asarray(sizes, dtype=np.int64)
    load = np.zeros(world, dtype=np.int64)
    owner = np.zeros(len(sizes), dtype=np.int64)
    for d in np.argsort(-sizes, kind="stable"):
        r = int(np.argmin(load))
        owner[d] = r
        load[r] += sizes[d]
    return [np.flatnonzero(owner == r) for r in range(world)]


def reduce_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduce one statistics block (int64[VR_STATS_WORDS]) across ranks; NCCL for CUDA
    tensors, gloo for CPU tensors.  The error word takes the minimum non-negative entry."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return stats.clone()
    s = stats.clone()
    summed = s.clone()
    dist.all_reduce(summed, op=dist.ReduceOp.SUM, group=group)
    maxed = s.clone()
    dist.all_reduce(maxed, op=dist.ReduceOp.MAX, group=group)
    err = s[N.VR_STAT_ERROR:N.VR_STAT_ERROR + 1].clone()
    big = torch.full_like(err, 2**62)
    err = torch.where(err < 0, big, err)
    dist.all_reduce(err, op=dist.ReduceOp.MIN, group=group)
    out = summed
    for w in MAX_WORDS:
        out[w] = maxed[w]
    out[N.VR_STAT_ERROR] = torch.where(err >= big, torch.full_like(err, -1), err)[0]
    return out
