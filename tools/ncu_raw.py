#!/usr/bin/env python3
"""Key raw metrics of one ncu capture (`ncu -i X --page raw --csv > f`):
stall reasons per issued instruction, pipe utilisation, memory counters."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units, vals = rows[0], rows[1], rows[2 if len(sys.argv) < 3 else 1 + int(sys.argv[2])]
d = {k: (v, u) for k, v, u in zip(h, vals, units)}
st = []
for k, (v, u) in d.items():
    if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('per_issue_active.ratio'):
        try:
            st.append((k, float(v.replace(',', ''))))
        except ValueError:
            pass
for k, v in sorted(st, key=lambda x: -x[1])[:12]:
    print('stall', k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), round(v, 2))
for k, (v, u) in sorted(d.items()):
    if ('pipe_' in k and 'pct_of_peak_sustained_active' in k and k.startswith('sm__')) or k in (
            'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
            'smsp__inst_executed.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
            'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'lts__t_sector_hit_rate.pct',
            'l1tex__t_sector_hit_rate.pct', 'launch__registers_per_thread',
            'sm__warps_active.avg.pct_of_peak_sustained_active'):
        try:
            if k.startswith('sm__') and 'pipe' in k and float(v.replace(',', '')) < 1:
                continue
        except ValueError:
            pass
        print(k, v, u)
