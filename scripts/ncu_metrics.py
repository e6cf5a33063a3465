#!/usr/bin/env python
"""Summarise an `ncu --metrics ... --csv --log-file X.csv` capture: per kernel, the mean of each
metric over its captured launches (time in us, DRAM bytes in MB, instructions in M)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("<")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
                 "Gbyte": 1e3, "inst": 1e-6, "cycle": 1e-3}.get(unit, 1.0)
        agg[(name, r[mi])].append(v * scale)
    for (name, m), vs in sorted(agg.items()):
        print(f"{name:32s} {m:36s} {sum(vs) / len(vs):12.3f}  (n={len(vs)})")


if __name__ == "__main__":
    main(sys.argv[1])
