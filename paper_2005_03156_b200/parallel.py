"""Multi-GPU plumbing: point shards, replicated index, histogram reduce.

The reference's only parallelism is ``run_chunked`` (parallel.hpp:30-82):
an atomic-cursor thread pool over fixed point chunks whose results are
concatenated in order.  Here the same decomposition runs one level up: each
GPU (one process per GPU, ``torch.distributed``) owns a contiguous shard of
the point stream, every rank builds the same index deterministically, and
ranks run independently -- each point's leaf depends only on the point and
the read-only index.  The one collective is the
optional per-block int64 point histogram (BASELINE config 5), summed with an
all-reduce every step: NCCL over NVLink on B200s, gloo in the CPU tests.

``bench.py`` runs :func:`run_steps` on every rank; ``tests/test_parallel_cpu.py``
runs the same function with two gloo ranks and the CPU oracle as projector.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Iterator, Optional

#: BASELINE config 5: 8B points over the whole job, split across the GPUs
C5_GLOBAL_POINTS = 8_000_000_000
#: most points one rank keeps resident per projection call (16 GB of points)
CHUNK_POINTS = 1 << 30


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
    if world < 1 or not (0 <= rank < world):
        raise ValueError("rank must be in [0, world)")
    return Shard(rank, world, rank * n_per_rank, n_per_rank)


@dataclass(frozen=True)
class Plan:
    """One rank's share of a projection job."""
    config: str
    shard: Shard
    scaling: str          # "weak": fixed points per GPU; "strong": fixed job
    global_points: int    # points projected by all ranks together per step
    chunk: int            # points resident at once on this rank
    hist: bool            # per-block histogram, all-reduced every step

    def chunks(self) -> Iterator[tuple[int, int]]:
        """(global offset, count) pieces of the shard, each <= chunk points."""
        off, end = self.shard.start, self.shard.start + self.shard.count
        while off < end:
            c = min(self.chunk, end - off)
            yield off, c
            off += c

    @property
    def resident(self) -> bool:
        """The whole shard fits one chunk: generated once, queried every step."""
        return self.shard.count <= self.chunk


def plan_workload(config: str, points: int, rank: int, world: int, hist: bool = False,
                  per_rank_default: Optional[int] = None, chunk: int = CHUNK_POINTS) -> Plan:
    """c5 is a fixed job of 8B points (``points`` overrides) split over the
    ranks -- strong scaling, histogram on.  Every other config gives each rank
    ``points`` (default: the config's own count) points of the stream --
    weak scaling; rank r owns the r-th slice."""
    if config == "c5":
        n_global = points or C5_GLOBAL_POINTS
        sh = shard_range(n_global, rank, world)
        return Plan(config, sh, "strong", n_global, max(1, min(chunk, sh.count)), True)
    per = points or per_rank_default
    if not per:
        raise ValueError("points per rank unknown")
    sh = weak_shard(per, rank, world)
    return Plan(config, sh, "weak", per * world, max(1, min(chunk, per)), hist)


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


def run_steps(plan: Plan, steps: int, project: Callable[[int, int], None],
              generate: Optional[Callable[[int, int], None]] = None,
              zero_hist: Optional[Callable[[], None]] = None,
              reduce: Optional[Callable[[], None]] = None,
              timed: Optional[Callable[[Callable[[], None]], None]] = None) -> None:
    """`steps` passes of this rank over its shard -- the per-rank loop of
    bench.py.  Per step: zero the histogram, project every chunk (a
    non-resident chunk is generated first, untimed), then reduce the
    histogram over the ranks.  ``project(offset, count)`` queries the chunk
    currently in the buffers; ``timed(fn)`` runs fn inside the timed
    accounting (default: plain call)."""
    run = timed or (lambda fn: fn())
    for _ in range(steps):
        if plan.hist and zero_hist is not None:
            run(zero_hist)
        for off, cnt in plan.chunks():
            if not plan.resident and generate is not None:
                generate(off, cnt)
            run(lambda off=off, cnt=cnt: project(off, cnt))
        if plan.hist and reduce is not None:
            run(reduce)
