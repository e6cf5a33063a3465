#!/usr/bin/env python
"""Per-CUDA-source-line executed instructions and stall samples from an ncu report
(cuda,sass correlated view): where the instructions and the stalls of a kernel come from."""
import collections
import csv
import io
import subprocess
import sys


def lines(rep, kernel_filter=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur_file, hdr, cur_line, cur_src = None, None, None, None
    agg = collections.defaultdict(lambda: [0, 0, ""])
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        # cuda-line rows have a line number in col 0; sass rows have an empty col 0
        if r[0].strip():
            cur_line, cur_src = r[0], r[1]
        try:
            ie = hdr.index("Instructions Executed")
            iss = hdr.index("Warp Stall Sampling (All Samples)")
            e = int(r[ie] or 0) if r[0].strip() else 0
            s = int(r[iss] or 0) if r[0].strip() else 0
        except (ValueError, IndexError):
            continue
        key = (cur_file, cur_line)
        agg[key][0] += e
        agg[key][1] += s
        agg[key][2] = cur_src
    return agg


if __name__ == "__main__":
    agg = lines(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    te = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total executed {te}, stall samples {ts}")
    byfile = collections.Counter()
    for (f, _), v in agg.items():
        byfile[f] += v[0]
    print({k: f"{100 * v / te:.1f}%" for k, v in byfile.items()})
    for (f, l), (e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * e / te:5.1f}% exec {100 * s / ts:5.1f}% stall  {f}:{l}  {src.strip()[:90]}")
    print("--- by stalls")
    for (f, l), (e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top // 2]:
        print(f"{100 * e / te:5.1f}% exec {100 * s / ts:5.1f}% stall  {f}:{l}  {src.strip()[:90]}")
