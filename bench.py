#!/usr/bin/env python3
"""Benchmark of the B200 point-to-block projection (BASELINE.json metric:
points projected/sec, device-timed, plus % of roofline, next to the
reference CPU path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
  python bench.py --impl reference ...      # the reference's CPU path

Default workload: BASELINE config 3 -- the largest config that fits one GPU
(12.5M-leaf nested tiling, 1B clustered points per GPU, 16 GB of points
resident in HBM next to the 47 GB index).  One step = one projection pass
(fm_query) over the rank's resident shard.  With --gpus N > 1 and no
torchrun environment, bench.py re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL); each rank owns a
contiguous shard of the global point stream and its own replica of the
index (parallel.py).  c5 is a fixed job of 8B points split over the ranks
(strong scaling) with the per-block int64 histogram all-reduced over NCCL
every step.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "points projected/sec (device-timed)"
UNIT = "points/s"

WORKLOADS = {
    "c3s": "c3s: 320,000-leaf nested hierarchy (10x5 states, 8x8 counties, 10x10 blocks, "
           "6 segs/edge), all three levels as FMCB, 100M clustered fp64 points",
    "c3mini": "c3mini: 40,000-leaf nested hierarchy (2x2 states, 4x4 counties, 25x25 blocks)",
    "c1": "c1: 1,024-polygon 32x32 jittered tiling (8 segs/edge, ~32 v), 1M uniform fp64 points",
    "c2": "c2: 250,000-polygon 500x500 jittered tiling (12 segs/edge, ~48 v), "
          "100M clustered fp64 points (2000 Zipf(1.1) centres, sigma 0.2 deg, 10% uniform)",
    "c4": "c4: 100,000-polygon 400x250 jittered tiling (50 segs/edge, sigma 0.15, ~200 v), "
          "200M fp64 points (50% uniform, 50% within 1e-4 cell of an edge)",
    "c3": "c3: 12.5M-leaf nested tiling (10x5 states, 20x20 counties, 25x25 blocks, 6 segs/edge), "
          "1B clustered fp64 points per GPU (20,000 Zipf(1.1) centres, 10% uniform)",
    "c5": "c5: the c3 index with 8B clustered points split over the GPUs + int64 per-block "
          "histogram all-reduced with NCCL every step",
}
# reference cover depth (best per config; c3/c5 at the
# deepest level whose single-threaded build fits the arm's few minutes:
# L16 = 134 s on the survey container, L18 did not finish in 10 min)
REF_MAX_LEVEL = {"c1": 12, "c2": 16, "c4": 16, "c3": 16, "c5": 16, "c3s": 16, "c3mini": 14}
# the in-bench cpu_baseline leg uses a quicker cover where the arm's takes minutes
CPU_LEG_MAX_LEVEL = {"c3": 14, "c5": 14}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--points", type=int, default=0,
                    help="points per GPU (c5: points of the whole job); default: the config's")
    ap.add_argument("--hist", action="store_true", help="also build the per-block int64 histogram")
    ap.add_argument("--mode", default="exact", choices=["exact", "approx", "simple", "simple-strict"],
                    help="CoverMode of the projection (approx: deemed leaves, error <= epsilon); "
                         "simple[-strict]: the hierarchical simple engine (nested configs)")
    ap.add_argument("--path", default="auto", choices=["auto", "stream", "binned"],
                    help="exact-mode query path (fm_index_set_query_path)")
    ap.add_argument("--epsilon", type=float, default=5e-3,
                    help="approx-mode cell diagonal bound in degrees")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-points", type=int, default=0,
                    help="points per rank in the e2e leg (default: the shard, <= 2^30 / N)")
    ap.add_argument("--check-points", type=int, default=100_000_000,
                    help="timed outputs checked against the CPU oracle per rank")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target seconds per CPU reference pass (bounded sample)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: run the multi-rank plumbing (gloo, CPU oracle as projector)")
    return ap.parse_args(argv)


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks, exactly as the driver launches it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(pathlib.Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, r in rows for k in range(4) if r[k] == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def cpu_reference_leg(cfg_name, soup, pts_host, threads, target_s, repeats=3, warmup=1,
                      max_level=None, one_thread=False):
    """Time the reference CPU path (oracle/_ref: query_leaves via run_chunked,
    F=4) on a bounded prefix of `pts_host`.  Returns a dict."""
    import oracle
    cores = threads or (os.cpu_count() or 1)
    level = max_level or REF_MAX_LEVEL[cfg_name]
    if oracle.ref_available():
        m = oracle.RefModel(soup)
        bi = m.build_index(level, 4)
        probe = pts_host[: min(len(pts_host), 500_000)]
        _, t = m.query_leaves(probe, threads=cores, want_ids=False)
        rate = len(probe) / max(t["seconds"], 1e-9)
        n = int(min(len(pts_host), max(len(probe), rate * target_s)))
        sample = np.ascontiguousarray(pts_host[:n])
        for _ in range(warmup):
            m.query_leaves(sample, threads=cores, want_ids=False)
        times = []
        for _ in range(repeats):
            _, t = m.query_leaves(sample, threads=cores, want_ids=False)
            times.append(t["seconds"])
        best = min(times)
        leg = {"value": n / best, "unit": UNIT, "cores": cores, "kind": "reference",
               "sample": f"first {n} points of this config's stream; reference "
                         f"query_leaves(exact) via run_chunked, cover max_level "
                         f"{level}, trie F=4; best of {repeats} after "
                         f"{warmup} warm-up (bench.hpp:82-94); cover build "
                         f"{bi['seconds']:.1f} s ({bi['entries']} entries) not counted",
               "times_s": times, "n": n, "max_level": level, "build_s": bi["seconds"]}
        if one_thread:  # also the 1-thread figure
            n1 = int(min(n, max(100_000, n // 16)))
            s1 = np.ascontiguousarray(pts_host[:n1])
            _, t1 = m.query_leaves(s1, threads=1, want_ids=False)
            leg["one_thread"] = {"value": n1 / t1["seconds"], "points": n1}
        return leg
    # oracle port (bucketed exhaustive_assign restatement) when _ref is absent
    probe = pts_host[: min(len(pts_host), 200_000)]
    t0 = time.perf_counter()
    oracle.assign(soup, probe, threads=cores)
    rate = len(probe) / max(time.perf_counter() - t0, 1e-9)
    n = int(min(len(pts_host), max(len(probe), rate * target_s)))
    sample = np.ascontiguousarray(pts_host[:n])
    times = []
    for _ in range(warmup + repeats):
        t0 = time.perf_counter()
        oracle.assign(soup, sample, threads=cores)
        times.append(time.perf_counter() - t0)
    best = min(times[warmup:])
    return {"value": n / best, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"first {n} points; oracle/oracle.c bucketed exhaustive_assign "
                      f"restatement (oracle/_ref absent)", "times_s": times[warmup:], "n": n}


_GEN_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2005_03156_b200 import synth
cfg = synth.config(sys.argv[2]); n = int(sys.argv[3]); out = sys.argv[4]
soup = cfg.make_soup()
np.save(out + "/vxy.npy", soup.vxy); np.save(out + "/ring_off.npy", soup.ring_off)
np.save(out + "/poly_ring.npy", soup.poly_ring)
pts = np.lib.format.open_memmap(out + "/pts.npy", mode="w+", dtype=np.float64, shape=(n, 2))
cfg.make_points(n, soup=soup, out=pts)
pts.flush()
"""


def run_reference(args):
    """The reference arm: the unmodified reference's query_leaves(exact) via
    run_chunked (oracle/_ref, compiled from /root/reference here), on all
    host threads, each step a bounded sample of this config's stream.  The
    inputs are generated by a separate process (the synth library never
    loads into this one)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2005_03156_b200.fastmap import Soup
    cores = os.cpu_count() or 1
    sample_n = min(args.points or 64_000_000, 64_000_000)
    with tempfile.TemporaryDirectory(prefix="fm_ref_") as tmp:
        subprocess.run([sys.executable, "-c", _GEN_SCRIPT, str(ROOT), args.config, str(sample_n), tmp],
                       check=True)
        soup = Soup(np.load(tmp + "/vxy.npy"), np.load(tmp + "/ring_off.npy"),
                    np.load(tmp + "/poly_ring.npy"))
        pts = np.load(tmp + "/pts.npy", mmap_mode="r")
        pts = np.ascontiguousarray(pts)
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    leg = cpu_reference_leg(args.config, soup, pts, cores, args.cpu_seconds,
                            repeats=max(1, args.steps), warmup=max(1, args.warmup), one_thread=True)
    step_s = statistics.mean(leg["times_s"])
    line = {
        "impl": "reference", "metric": METRIC, "value": leg["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(leg["times_s"]), "warmup": max(1, args.warmup),
        "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c5" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "sample_points": leg["n"],
                   "same_config": True,
                   "sample": "the first points of the same seeded stream our arm projects "
                             "(host generator = device generator bit for bit)",
                   "parallelism": f"host threads (run_chunked), {cores} cores",
                   "ref_max_level": leg.get("max_level"), "ref_cover_build_s": leg.get("build_s")},
        "cpu_baseline": {k: leg[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "cpu_one_thread": leg.get("one_thread"),
        "e2e": {"value": leg["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_ours(args):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2005_03156_b200 import fastmap, parallel, synth

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    host_threads = max(1, (os.cpu_count() or 1) // world)

    cfg = synth.config(args.config)
    plan = parallel.plan_workload(args.config, args.points, rank, world, hist=args.hist,
                                  per_rank_default=cfg.n_points)
    soup = cfg.make_soup(threads=host_threads)
    approx = args.mode == "approx"
    mode = fastmap.CoverMode.approx if approx else fastmap.CoverMode.exact
    params = (fastmap.CoverParams(mode=mode, epsilon=args.epsilon, threads=host_threads) if approx
              else fastmap.CoverParams(threads=host_threads))
    t0 = time.perf_counter()
    idx = fastmap.build_index(soup, params, device=local)
    build_s = time.perf_counter() - t0
    idx.set_query_path(args.path)
    st = idx.stats()
    qplan = idx.query_plan(plan.chunk)

    d_pts = torch.empty((plan.chunk, 2), dtype=torch.float64, device=dev)
    d_out = torch.empty(plan.chunk, dtype=torch.int32, device=dev)
    d_hist = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev) if plan.hist else None
    stream = torch.cuda.current_stream(dev)
    soup_dev = None
    if getattr(cfg, "points", "") == "near_edge":
        soup_dev = (torch.from_numpy(soup.vxy).to(dev),
                    torch.from_numpy(soup.ring_off.view(np.int64)).to(dev),
                    torch.from_numpy(soup.poly_ring.view(np.int64)).to(dev))

    def generate(off, cnt):
        cfg.make_points_device(d_pts[:cnt], offset=off, soup=soup, stream=stream, soup_device=soup_dev)

    def project(off, cnt):
        idx.project(d_pts[:cnt], out=d_out[:cnt], hist=d_hist, stream=stream, mode=mode)

    def zero_hist():
        d_hist.zero_()

    def reduce():
        parallel.reduce_histogram(d_hist)

    if plan.resident:
        generate(plan.shard.start, plan.shard.count)
    torch.cuda.synchronize()
    warm = max(3, args.warmup)
    parallel.run_steps(plan, warm, project, generate, zero_hist, reduce)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    pairs = []

    def timed(fn):  # CUDA events on the launching stream around each timed call
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        pairs.append((e0, e1))

    with ClockSampler(local) as clk:
        if plan.resident:  # one event pair around all K steps
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            parallel.run_steps(plan, args.steps, project, generate, zero_hist, reduce)
            e1.record(stream)
            pairs.append((e0, e1))
        else:  # chunks regenerated between projections: only the projections are timed
            parallel.run_steps(plan, args.steps, project, generate, zero_hist, reduce, timed=timed)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in pairs)
    ms_max = parallel.max_over_ranks(ms, device=dev)
    value = plan.global_points * args.steps / (ms_max / 1e3)
    launch_ms = ms / args.steps / max(1, sum(1 for _ in plan.chunks()))

    # parity: the timed output (last chunk of the last step) against the CPU oracle
    last_off, last_cnt = list(plan.chunks())[-1]
    n_chk = int(min(last_cnt, args.check_points))
    if n_chk < last_cnt:
        sel = torch.from_numpy(np.sort(np.random.default_rng(rank).choice(
            last_cnt, size=n_chk, replace=False))).to(dev)
        chk_pts, got = d_pts[:last_cnt][sel].cpu().numpy(), d_out[:last_cnt][sel].cpu().numpy()
    else:
        chk_pts, got = d_pts[:last_cnt].cpu().numpy(), d_out[:last_cnt].cpu().numpy()
    t0 = time.perf_counter()
    want = oracle.assign(soup, chk_pts, threads=host_threads)
    chk_s = time.perf_counter() - t0
    mismatches = int((got != want).sum())
    parity = {"checked_points": int(n_chk), "mismatches_vs_oracle": mismatches,
              "of_points": int(last_cnt), "oracle_s": round(chk_s, 2)}
    if approx:  # disagreements are allowed within epsilon (test_cell_index.cpp:381-435)
        far = 0
        for k in np.nonzero(got != want)[0][:2000]:
            p = chk_pts[k]
            far += int(got[k] < 0 or oracle.point_polygon_distance(
                soup, int(got[k]), float(p[0]), float(p[1])) > args.epsilon)
        parity = {"checked_points": int(n_chk), "approx_disagreements": mismatches,
                  "beyond_epsilon": far, "epsilon": args.epsilon}
        mismatches = far
    hist_check = None
    if plan.hist:  # the reduced histogram counts every point of the job exactly once
        tot = int(d_hist.sum().item())
        hist_check = {"total": tot, "assigned_in_check_sample": int((want >= 0).sum())}
    del chk_pts, got, want

    # e2e: the public host-buffer API (fm_query_host), H2D and D2H inside the region
    e2e = None
    if not args.no_e2e:
        ne = int(min(last_cnt, args.e2e_points or max(1, (1 << 30) // world)))
        ph = torch.empty((ne, 2), dtype=torch.float64, pin_memory=True)
        ph.copy_(d_pts[:ne])
        oh = torch.empty(ne, dtype=torch.int32, pin_memory=True)
        hist_h = np.zeros(soup.n_polys, dtype=np.int64) if plan.hist else None
        ph_np, oh_np = ph.numpy(), oh.numpy()
        idx.project(ph_np, out=oh_np, hist=hist_h, mode=mode)  # warm (allocates staging)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            idx.project(ph_np, out=oh_np, hist=hist_h, mode=mode)
        el = parallel.max_over_ranks(time.perf_counter() - t0, device=dev)
        e2e_ok = bool(np.array_equal(oh_np, d_out[:ne].cpu().numpy()))
        e2e = {"value": ne * world * args.e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": 16 * ne * world, "d2h_bytes_per_step": 4 * ne * world,
               "points_per_rank": ne, "equal_to_device_path": e2e_ok,
               "path": "fm_query_host (pinned host buffers, 3-stream chunked H2D/kernel/D2H)"}
        del ph, oh

    cpu = None
    if rank == 0 and not args.no_cpu:
        ncpu = int(min(last_cnt, 64_000_000))
        host = d_pts[:ncpu].cpu().numpy()
        leg = cpu_reference_leg(args.config, soup, host, os.cpu_count() or 1, args.cpu_seconds,
                                max_level=CPU_LEG_MAX_LEVEL.get(args.config))
        cpu = {k: leg[k] for k in ("value", "unit", "cores", "kind", "sample")}
        del host

    peak, peak_kind = measured_peaks()
    npl = plan.chunk  # points per projection call
    alg_bytes = 20.0 * npl + 16.0 * soup.n_vertices  # SURVEY.md sec. 8d per-point + index once
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / (f"ncu_{args.config}_approx_summary.json" if approx
                                else f"ncu_{args.config}_summary.json")
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    binned = (not approx) and qplan["path"] == "binned"
    # our kernels per fm_query call (fastmap_b200.cu launch()): the stream
    # path runs stream_kernel + resolve_kernel per 2^28-point slice, the
    # binned path sample + plan + scatter + seal + query + unbin + unplaced
    # per 2^30-point batch, approx one kernel; with a histogram, one
    # widen_hist_kernel per slice / batch (and binned_hist_kernel per batch)
    launches_per_call = []
    for _, cnt in plan.chunks():
        if approx:
            launches_per_call.append(1 + (1 if plan.hist else 0))
        else:
            unit = (1 << 30) if binned else (1 << 28)
            pieces = -(-cnt // unit)
            launches_per_call.append(pieces * ((7 if binned else 2)
                                               + ((2 if binned else 1) if plan.hist else 0)))
    n_launches = args.steps * sum(launches_per_call)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": plan.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe, generated on the GPU; DESIGN.md sec. 3)",
            "config": {
                "workload": WORKLOADS[args.config], "points_per_gpu": plan.shard.count,
                "global_points": plan.global_points, "polygons": soup.n_polys,
                "vertices": soup.n_vertices, "histogram": plan.hist, "mode": args.mode,
                "epsilon": args.epsilon if approx else None,
                "parallelism": f"point shards x{world} (NCCL), index replicated",
                "resident": plan.resident, "points_per_call": npl,
                "l2": "inputs larger than L2 (16 B/pt stream), no flush",
                "index": {k: st[k] for k in ("nx", "ny", "cells_hit", "cells_boundary",
                                             "grid_bytes", "arena_bytes", "query_grid_bytes",
                                             "query_block_log2", "approx_grid_bytes",
                                             "approx_block_log2", "slots_total", "slots_double",
                                             "cells_split", "build_phase_seconds")},
                "index_build_s": build_s,
                "query_path": None if approx else qplan,
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_kind,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel": ("fm_query_mode(approx) = approx_kernel" if approx else
                                    "fm_query = bin_sample + bin_plan + bin_scatter + bin_seal + binned_query + unbin + unplaced"
                                    if binned else "fm_query = stream_kernel + resolve_kernel"),
                         "launch_ms": launch_ms,
                         "traffic_source": "profiles/%s (ncu, cold cache)" % prof.name},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_launches,
            "clocks": clk.summary(),
            "parity": parity,
            "histogram_check": hist_check,
        }
        print(json.dumps(line), flush=True)
    idx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0 if mismatches == 0 else 3


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU -- gloo ranks, the
    same plan / run_steps / histogram reduce as run_ours, the CPU oracle as
    the projector on a small stream.  Prints a line with "dry_run": true."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2005_03156_b200 import parallel, synth

    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    name = "c1" if args.config in ("c3", "c5", "c3s") else args.config
    cfg = synth.config(name)
    soup = cfg.make_soup()
    n_job = args.points or 200_000
    plan = parallel.plan_workload(args.config if args.config == "c5" else name, n_job, rank, world,
                                  hist=args.hist, per_rank_default=cfg.n_points, chunk=50_000)
    hist = torch.zeros(soup.n_polys, dtype=torch.int64)
    buf = {}

    def generate(off, cnt):
        buf["pts"] = cfg.make_points(cnt, offset=off, soup=soup)

    def project(off, cnt):
        if plan.resident and "pts" not in buf:
            generate(off, cnt)
        ids = oracle.assign(soup, buf["pts"], threads=1)
        if plan.hist:
            hist.add_(torch.from_numpy(np.bincount(ids[ids >= 0], minlength=soup.n_polys)))

    t0 = time.perf_counter()
    parallel.run_steps(plan, args.steps, project, generate, lambda: hist.zero_(),
                       lambda: parallel.reduce_histogram(hist))
    el = parallel.max_over_ranks(time.perf_counter() - t0)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "scaling": plan.scaling,
                          "config": {"workload": WORKLOADS.get(args.config), "stand_in": name,
                                     "global_points": plan.global_points,
                                     "points_per_rank": plan.shard.count,
                                     "chunks_per_rank": sum(1 for _ in plan.chunks())},
                          "histogram_total": int(hist.sum().item()) if plan.hist else None,
                          "wall_s": el}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_simple(args):
    """The simple engine (simple_mapper.hpp:119-166) on one nested config:
    one step = assign() of the rank's resident points (one kernel)."""
    import tempfile

    import torch
    import torch.distributed as dist

    from paper_2005_03156_b200 import fastmap, synth

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    cfg = synth.config(args.config)
    if not hasattr(cfg, "write_fmcb"):
        raise SystemExit("--mode simple needs a nested config (c3s, c3mini, c3)")
    mode = fastmap.AssignMode.strict if args.mode == "simple-strict" else fastmap.AssignMode.relaxed
    n = args.points or cfg.n_points
    pts_host = torch.empty((n, 2), dtype=torch.float64, pin_memory=True)
    cfg.make_points(n, offset=rank * n, out=pts_host.numpy())
    fd, path = tempfile.mkstemp(suffix=".fmcb")
    os.close(fd)
    t0 = time.perf_counter()
    cfg.write_fmcb(path)
    h = fastmap.load_hierarchy(path)
    eng = fastmap.SimpleEngine(h, local)
    build_s = time.perf_counter() - t0
    d_pts = pts_host.to(dev)
    outs = tuple(torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3))
    stream = torch.cuda.current_stream(dev)

    def step():
        eng.assign(d_pts, mode, counters=False, out=outs, stream=stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # parity: the reference's own assign() on the same FMCB bytes (oracle/_ref)
    import oracle
    chk = np.random.default_rng(rank).choice(n, size=min(n, 20_000), replace=False)
    parity = {"checked_points": int(len(chk))}
    if oracle.ref_available():
        st, co, bl, _ = oracle.ref_simple_assign(path, pts_host.numpy()[chk],
                                                 mode == fastmap.AssignMode.strict)
        got = [o.cpu().numpy()[chk] for o in outs]
        parity["mismatches_vs_reference"] = int(((got[0] != st) | (got[1] != co) |
                                                 (got[2] != bl)).sum())
    e2e = None
    if not args.no_e2e:
        ph = pts_host.numpy()
        eng.assign(ph[: min(n, 1 << 20)], mode, counters=False)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            eng.assign(ph, mode, counters=False)
        el = time.perf_counter() - t0
        e2e = {"value": n * world * args.e2e_steps / el, "unit": UNIT,
               "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 12 * n,
               "path": "fm_simple_assign_host (8M-point chunks)"}
    os.unlink(path)
    peak, peak_kind = measured_peaks()
    launch_ms = ms / args.steps
    alg_bytes = 28.0 * n + 16.0 * (h.soup.n_vertices)  # 16 B in + 3 x 4 B out per point
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": n * world * args.steps / (ms_max / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE recipe; see DESIGN.md sec. 3)",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "mode": args.mode,
                       "points_per_gpu": n, "global_points": n * world,
                       "states": int(h.n_states), "counties": int(h.n_counties),
                       "blocks": int(h.n_leaves), "parallelism": f"point shards x{world}",
                       "l2": "inputs larger than L2 (16 B/pt stream), no flush",
                       "engine_build_s": build_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel": "fm_simple_assign = simple_kernel", "launch_ms": launch_ms},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": args.steps,
            "clocks": clk.summary(), "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity.get("mismatches_vs_reference", 0) == 0 else 3


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    if args.mode in ("simple", "simple-strict"):
        return run_simple(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
