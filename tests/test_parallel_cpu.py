"""Multi-rank host logic on CPU (gloo, world_size 2): point sharding and the
per-block histogram reduce that config 5 runs over NCCL on B200s.  The
per-rank ids come from the CPU oracle here (no GPU in this container); the
sharding / reduction code is the same the GPU ranks run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_03156_b200 import parallel, synth


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            shards = [parallel.shard_range(n, r, w) for r in range(w)]
            assert sum(s.count for s in shards) == n
            pos = 0
            for s in shards:
                assert s.start == pos
                pos += s.count
            assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
    with pytest.raises(ValueError):
        parallel.shard_range(10, 2, 2)


def test_weak_shards_are_disjoint_stream_slices():
    cfg = synth.config("c1")
    a = cfg.make_points(1000, offset=parallel.weak_shard(1000, 1, 2).start)
    full = cfg.make_points(2000)
    assert np.array_equal(a, full[1000:])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_global, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    sh = parallel.shard_range(n_global, rank, world)
    pts = cfg.make_points(sh.count, offset=sh.start)
    ids = oracle.assign(soup, pts, threads=1)
    hist = torch.from_numpy(np.bincount(ids[ids >= 0], minlength=soup.n_polys).astype(np.int64))
    parallel.reduce_histogram(hist)
    t = parallel.max_over_ranks(float(rank + 1))
    out_q.put((rank, hist.numpy(), t))
    dist.barrier()
    dist.destroy_process_group()


def test_histogram_allreduce_two_ranks_matches_single_process():
    n_global = 20_000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_global, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    ids = oracle.assign(soup, cfg.make_points(n_global))
    want = np.bincount(ids[ids >= 0], minlength=soup.n_polys)
    for rank, hist, t in res:
        assert np.array_equal(hist, want), f"rank {rank} histogram differs"
        assert t == 2.0  # max over ranks
