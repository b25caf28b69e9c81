#!/usr/bin/env python3
"""Per-fm_query summary of an ncu launch list (gpu__time_duration.sum,
dram__bytes_read/write.sum[, lts__t_bytes.sum] per launch, cold cache,
serialised), for a run of `calls` fm_query calls of `points` points each:

  python tools/summarize_launches.py LAUNCHES.csv CALLS POINTS CONFIG OUT.json

Writes OUT.json; its `dram_bytes_per_launch` (DRAM bytes of one fm_query
call, all its kernels) is what bench.py reports as roofline.traffic."""
import csv
import json
import sys
from collections import defaultdict

path, calls, points, config, out = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4], sys.argv[5]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = defaultdict(lambda: defaultdict(float))
nl = defaultdict(set)
for r in rows[1:]:
    k = r[ki].split("(")[0].split("::")[-1].split("<")[0].strip()
    per[k][r[mi]] += float(r[vi].replace(",", ""))
    nl[k].add(r[0])
summ = {"config": config, "points_per_call": points, "calls": calls,
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
                  f" --clock-control none ({path.split('/')[-1]}); per fm_query call = total / calls"}
tot_b = tot_ns = 0.0
for k, m in per.items():
    d = {"launches_per_call": len(nl[k]) / calls,
         "ns_per_call": m["gpu__time_duration.sum"] / calls,
         "dram_read_bytes_per_call": m["dram__bytes_read.sum"] / calls,
         "dram_write_bytes_per_call": m["dram__bytes_write.sum"] / calls}
    if "lts__t_bytes.sum" in m:
        d["l2_bytes_per_call"] = m["lts__t_bytes.sum"] / calls
    d["dram_bytes_per_call"] = d["dram_read_bytes_per_call"] + d["dram_write_bytes_per_call"]
    summ[k] = d
    tot_b += d["dram_bytes_per_call"]
    tot_ns += d["ns_per_call"]
for k in per:
    summ[k]["share_of_fm_query"] = summ[k]["ns_per_call"] / tot_ns
summ["dram_bytes_per_launch"] = tot_b
summ["dram_bytes_per_point"] = tot_b / points
summ["fm_query_ns_ncu"] = tot_ns
open(out, "w").write(json.dumps(summ, indent=1) + "\n")
print(json.dumps(summ, indent=1))
