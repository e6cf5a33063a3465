#!/usr/bin/env python
"""Turn a gpurun ncu capture (full report + launch list) into the committed profiles/ summary:
profiles/<tag>_step_ncu.txt (metrics + hottest lines), profiles/<tag>_launches.txt (per-kernel
share of the launch list) and profiles/ncu_step_summary.json (per-launch DRAM traffic read by
bench.py's roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import ncu_lines  # noqa: E402
import ncu_summary  # noqa: E402


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    k, m, v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hdr_i + 1:]:
        if len(r) <= v:
            continue
        name = r[k].split("(")[0]
        per[name][r[m]].append(float(r[v].replace(",", "")))
    return per


def main(tag, rep, launch_csv, workload, n_env):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = []
    for d in ncu_summary.raw(rep):
        lines.append(d.pop("kernel")[:140])
        for key, (val, unit) in d.items():
            lines.append(f"  {key:80s} {val} {unit}")
    lines += ncu_summary.hot_sass(rep, top=20)
    agg = ncu_lines.lines(rep)
    te = sum(x[0] for x in agg.values()) or 1
    ts = sum(x[1] for x in agg.values()) or 1
    lines.append("hottest CUDA source lines (executed %, stall %):")
    for (f, ln), (e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        lines.append(f"  {100 * e / te:5.1f}% {100 * s / ts:5.1f}%  {f}:{ln}  {src.strip()[:100]}")
    with open(os.path.join(ROOT, "profiles", f"{tag}_step_ncu.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    per = launches(launch_csv)
    tot = sum(sum(mm.get("gpu__time_duration.sum", [])) for mm in per.values()) or 1
    out = [f"launch list ({launch_csv}): ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
           f"dram__bytes_write.sum --clock-control none (cold-cache, serialised: compare shares)"]
    step = None
    for name, mm in sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = mm.get("gpu__time_duration.sum", [])
        rd, wr = mm.get("dram__bytes_read.sum", []), mm.get("dram__bytes_write.sum", [])
        share = 100 * sum(t) / tot
        out.append(f"  {name[:90]:90s} launches {len(t):3d}  share {share:5.1f}%  mean {sum(t) / max(len(t), 1) / 1e3:8.1f} us"
                   + (f"  dram/launch {(sum(rd) + sum(wr)) / max(len(rd), 1) / 1e6:8.1f} MB" if rd else ""))
        if "step_kernel" in name and rd:
            step = (sum(rd) + sum(wr)) / len(rd)
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    js_path = os.path.join(ROOT, "profiles", "ncu_step_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    # the units of ncu's raw export are MB/KB-scaled: take dram bytes from the full capture instead
    full = ncu_summary.raw(rep)[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb = float(full["dram__bytes_read.sum"][0]) * scale.get(full["dram__bytes_read.sum"][1], 1)
    wb = float(full["dram__bytes_write.sum"][0]) * scale.get(full["dram__bytes_write.sum"][1], 1)
    js[workload] = {"tag": tag, "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                    "n_env": n_env, "bytes_per_env": (rb + wb) / n_env,
                    "launch_list_dram_bytes_per_launch": step}
    json.dump(js, open(js_path, "w"), indent=1)
    print("\n".join(lines[:40]))
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "cfg4-1M-envs-full-pipeline",
         int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 20)
