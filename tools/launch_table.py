#!/usr/bin/env python3
"""Per-kernel mean duration / DRAM bytes from an ncu launch list (csv):
  python tools/launch_table.py launches.csv [skip_first_n_launches_per_kernel]"""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iM, iV, iU, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    k = r[iK].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    d.setdefault((r[iID], k), {})[r[iM]] = float(r[iV].replace(",", "")) * (1e3 if r[iU] in ("us", "usecond") else 1e6 if r[iU] in ("ms", "msecond") else 1)
agg = collections.OrderedDict()
for (i, k), m in d.items():
    agg.setdefault(k, []).append(m)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, ms in agg.items():
    ms = ms[skip:] or ms
    t = sum(x.get("gpu__time_duration.sum", 0) for x in ms) / len(ms)
    rd = sum(x.get("dram__bytes_read.sum", 0) for x in ms) / len(ms)
    wr = sum(x.get("dram__bytes_write.sum", 0) for x in ms) / len(ms)
    l2 = sum(x.get("lts__t_bytes.sum", 0) for x in ms) / len(ms)
    print(f"{k[:44]:44s} n={len(ms):3d}  {t/1e6:8.3f} ms  rd {rd/1e9:7.2f} GB  wr {wr/1e9:7.2f} GB  l2 {l2/1e9:7.2f} GB  {(rd+wr)/max(t,1):6.2f} TB/s" .replace("TB/s","GB/ms"))
