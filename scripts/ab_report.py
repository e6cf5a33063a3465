#!/usr/bin/env python
"""Summarise gpurun_out/ab_*.log bench lines: variant -> value, ms/step, roofline frac, clocks."""
import glob
import json
import os
import sys

rows = []
for f in sorted(glob.glob(os.path.join(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out", "ab_*.log"))):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            r = d.get("roofline") or {}
            c = d.get("clocks") or {}
            rows.append((os.path.basename(f)[3:-4], d["value"], d["ms_per_step"], r.get("frac"), c.get("sm_mhz"),
                         ",".join(c.get("reasons") or [])))
for r in rows:
    print(f"{r[0]:24s} {r[1]:.4g} {r[2]:.4f} ms  frac {r[3]:.3f}  sm {r[4]}  {r[5]}")
