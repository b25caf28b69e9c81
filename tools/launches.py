#!/usr/bin/env python3
"""Mean per-kernel metrics of an ncu --csv launch list."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
d = defaultdict(list)
for r in rows[1:]:
    d[(r[ki].split('(')[0].split('::')[-1], r[mi])].append(float(r[vi].replace(',', '')))
for k, v in sorted(d.items()):
    print(k[0].ljust(36), k[1].ljust(32), len(v), round(sum(v) / len(v), 4))
