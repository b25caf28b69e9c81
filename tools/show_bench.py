#!/usr/bin/env python3
"""One line per bench log: python tools/show_bench.py LOG [LOG ...]"""
import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{"metric"') or l.startswith('{"impl"'):
            d = json.loads(l)
            c = d.get("config", {})
            print(f.split("/")[-1], "|", c.get("workload", "")[:12], "| value %.3e" % d["value"], "| ms %.3f" % d.get("ms_per_step", 0),
                  "| frac", round((d.get("roofline") or {}).get("frac", 0), 4), "| e2e", (d.get("e2e") or {}).get("value"),
                  "| cpu", (d.get("cpu_baseline") or {}).get("value"), "| parity", d.get("parity"), "| hist", d.get("histogram_check"),
                  "| path", (c.get("query_path") or {}), "| clocks", d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
