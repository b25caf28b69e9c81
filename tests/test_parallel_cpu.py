"""Multi-rank host logic on CPU (gloo, world_size 2): the per-rank loop
bench.py runs on every GPU (parallel.plan_workload + parallel.run_steps),
with the per-block histogram all-reduced every step -- NCCL over NVLink on
B200s, gloo here.  The projector is the CPU oracle in these tests (no GPU
in this container); the sharding, chunking and reduction code is the one
the GPU ranks run."""
import os
import pathlib
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


def _worker(rank, world, port, config, n_points, chunk, steps, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    plan = parallel.plan_workload(config, n_points, rank, world, hist=True,
                                  per_rank_default=cfg.n_points, chunk=chunk)
    hist = torch.zeros(soup.n_polys, dtype=torch.int64)
    buf, ids_out = {}, {}

    def generate(off, cnt):
        buf["pts"] = cfg.make_points(cnt, offset=off)

    def project(off, cnt):
        if "pts" not in buf:  # resident shard: generated once
            generate(off, cnt)
        ids = oracle.assign(soup, buf["pts"], threads=1)
        ids_out[off] = ids
        hist.add_(torch.from_numpy(np.bincount(ids[ids >= 0], minlength=soup.n_polys)))

    parallel.run_steps(plan, steps, project, generate, lambda: hist.zero_(),
                       lambda: parallel.reduce_histogram(hist))
    t = parallel.max_over_ranks(float(rank + 1))
    ids = np.concatenate([ids_out[k] for k in sorted(ids_out)])
    out_q.put((rank, plan.shard.start, ids, hist.numpy(), t, plan.scaling, plan.global_points))
    dist.barrier()
    dist.destroy_process_group()


def _run_two_ranks(config, n_points, chunk, steps=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, config, n_points, chunk, steps, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("config,n_points,chunk", [("c5", 30_001, 7_000),   # strong, chunked
                                                   ("c1", 12_000, 1 << 30)])  # weak, resident
def test_two_ranks_run_steps_match_one_process(config, n_points, chunk):
    """Both ranks' outputs, concatenated in rank order, equal the single-
    process answers on the whole job; the reduced histogram after every
    step counts every point of the job exactly once on every rank; the
    timing reduce takes the max over ranks."""
    import oracle
    res = _run_two_ranks(config, n_points, chunk)
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    n_global = res[0][6]
    assert n_global == (n_points if config == "c5" else 2 * n_points)
    assert res[0][5] == ("strong" if config == "c5" else "weak")
    ids = oracle.assign(soup, cfg.make_points(n_global))
    assert res[0][1] == 0 and res[1][1] == len(res[0][2])
    assert np.array_equal(np.concatenate([r[2] for r in res]), ids)
    want = np.bincount(ids[ids >= 0], minlength=soup.n_polys)
    for rank, _, _, hist, t, _, _ in res:
        assert np.array_equal(hist, want), f"rank {rank} histogram differs"
        assert t == 2.0  # max over ranks


def test_plan_chunks_cover_the_shard():
    p = parallel.plan_workload("c5", 10_000_000_019, 3, 8, chunk=1 << 30)
    assert p.scaling == "strong" and p.hist and p.global_points == 10_000_000_019
    pieces = list(p.chunks())
    assert pieces[0][0] == p.shard.start and sum(c for _, c in pieces) == p.shard.count
    assert all(c <= 1 << 30 for _, c in pieces) and not p.resident
    q = parallel.plan_workload("c3", 0, 1, 4, per_rank_default=1_000_000_000)
    assert q.scaling == "weak" and q.shard.start == 1_000_000_000 and q.resident
    assert q.global_points == 4_000_000_000 and not q.hist


def test_bench_dry_run_two_ranks_reports_n_gpus():
    """bench.py --gpus 2 re-launches itself under torch.distributed.run with
    two ranks; the dry run (gloo, CPU oracle) must report n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = pathlib.Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--dry-run", "--gpus", "2",
                        "--config", "c5", "--steps", "2", "--points", "120000"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["dry_run"] and line["scaling"] == "strong"
    assert line["config"]["global_points"] == 120000 and line["config"]["points_per_rank"] == 60000
