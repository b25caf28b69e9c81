"""Multi-GPU plumbing: point shards, replicated index, histogram reduce.

The projection has no data-path exchange: each point's
leaf depends only on the point and the read-only index, so points are
sharded by contiguous index ranges across ranks (one process per GPU), every
rank builds (deterministically) its own replica of the index, and ranks run
independently.  The only collective is the optional per-block int64 point
histogram (BASELINE config 5), summed with one all-reduce -- NCCL over
NVLink on B200s, gloo in the CPU tests.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int   # first global point index of this rank
    count: int   # points owned by this rank


def shard_range(n_global: int, rank: int, world: int) -> Shard:
    """Contiguous, balanced split of [0, n_global): the first n_global % world
    ranks get one extra point.  Shards are disjoint and cover everything."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank must be in [0, world)")
    if n_global < 0:
        raise ValueError("n_global must be >= 0")
    base, extra = divmod(n_global, world)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, base + (1 if rank < extra else 0))


def weak_shard(n_per_rank: int, rank: int, world: int) -> Shard:
    """Weak scaling: every rank owns n_per_rank points of the global stream."""
    return Shard(rank, world, rank * n_per_rank, n_per_rank)


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def reduce_histogram(hist, group=None):
    """Sum per-block point counts over all ranks in place (torch tensor,
    int64).  On CUDA tensors this is one NCCL all-reduce over NVLink."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timing: a multi-GPU step is as slow as
    its slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class ShardedProjector:
    """One rank's view of a sharded projection: a replica of the index on
    this rank's GPU, projecting this rank's point shard."""

    def __init__(self, soup, params=None, device: Optional[int] = None):
        from . import fastmap
        rank, world, local = dist_env()
        self.rank, self.world = rank, world
        self.device = local if device is None else device
        self.index = fastmap.build_index(soup, params, device=self.device)
        self.n_leaves = soup.n_polys

    def project(self, points, out=None, hist=None, stream=None):
        return self.index.project(points, out=out, hist=hist, stream=stream)

    def histogram(self, ids) -> np.ndarray:
        """Host helper: per-leaf counts of an id array (tests / reports)."""
        ids = np.asarray(ids)
        return np.bincount(ids[ids >= 0], minlength=self.n_leaves).astype(np.int64)

    def close(self):
        self.index.close()
