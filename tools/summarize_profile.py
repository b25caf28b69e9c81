#!/usr/bin/env python3
"""Turn a round's ncu artefacts (gpurun_out/launches_<tag>.csv and
prof_<tag>.ncu-rep) into committed summaries under profiles/<tag>/:
  launches.csv      the per-launch device-time / DRAM list (ncu, cold, serialised)
  summary.json      per-kernel mean duration and DRAM bytes per launch, and the
                    per-fm_query total bench.py reports as roofline.traffic
  details_<k>.txt   key metrics of the full capture of each kernel
and copy summary.json to profiles/ncu_<config>_summary.json (read by bench.py)."""
import csv
import io
import json
import pathlib
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = pathlib.Path(__file__).resolve().parent.parent


def kernel_name(full: str) -> str:
    """'void <unnamed>::stream_kernel<0, 0>(...)' -> 'stream_kernel'"""
    head = full.split("(")[0]
    head = head.split("<0")[0].split("<1")[0]
    return head.split("::")[-1].strip()


def main(tag, config="c2", points=100_000_000, mode="exact"):
    """mode "approx": gpurun_out/launches_approx_<tag>.csv (approx_kernel) ->
    profiles/<tag>/approx_summary.json and profiles/ncu_<config>_approx_summary.json."""
    out = ROOT / "profiles" / tag
    out.mkdir(parents=True, exist_ok=True)
    sfx = "" if mode == "exact" else "approx_"
    lcsv = ROOT / "gpurun_out" / f"launches_{sfx}{tag}.csv"
    rows = [r for r in csv.reader(open(lcsv)) if len(r) > 10 and r[0] != "ID"]
    per = defaultdict(lambda: defaultdict(list))
    for r in rows:
        kname = kernel_name(r[4])
        per[kname][r[-3]].append(float(r[-1]))
    summ = {"config": config, "points_per_launch": points, "source": "ncu --metrics "
            "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"}
    total_bytes = 0.0
    total_ns = 0.0
    for k, m in per.items():
        n = len(m["gpu__time_duration.sum"])
        d = {"launches": n,
             "mean_ns": sum(m["gpu__time_duration.sum"]) / n,
             "dram_read_bytes": sum(m["dram__bytes_read.sum"]) / n,
             "dram_write_bytes": sum(m["dram__bytes_write.sum"]) / n}
        d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        summ[k] = d
        total_bytes += d["dram_bytes"]
        total_ns += d["mean_ns"]
    summ["dram_bytes_per_launch"] = total_bytes
    summ["dram_bytes_per_point"] = total_bytes / points
    summ["fm_query_ns_ncu"] = total_ns
    for k in per:
        summ[k]["share_of_fm_query"] = summ[k]["mean_ns"] / total_ns
    shutil.copy(lcsv, out / f"launches{'' if mode == 'exact' else '_approx'}.csv")
    rep = ROOT / "gpurun_out" / f"prof_{tag}.ncu-rep"
    if rep.exists() and mode == "exact":
        txt = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"],
                             capture_output=True, text=True).stdout
        by_k = defaultdict(list)
        for d in csv.DictReader(io.StringIO(txt)):
            k = kernel_name(d.get("Kernel Name", ""))
            by_k[k].append(f"{d['Section Name'][:34]:34s} {d['Metric Name'][:52]:52s} "
                           f"{d['Metric Value']} {d['Metric Unit']}")
        for k, lines in by_k.items():
            (out / f"details_{k}.txt").write_text("\n".join(lines) + "\n")
    name = "summary.json" if mode == "exact" else "approx_summary.json"
    (out / name).write_text(json.dumps(summ, indent=1) + "\n")
    shutil.copy(out / name, ROOT / "profiles" / (f"ncu_{config}_summary.json" if mode == "exact"
                                                 else f"ncu_{config}_approx_summary.json"))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], mode=sys.argv[2] if len(sys.argv) > 2 else "exact")
