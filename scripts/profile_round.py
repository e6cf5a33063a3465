#!/usr/bin/env python
"""Commit one gpurun evidence run (scripts/gpu_round2_final.sh, prefix gpurun_out/<run>_) into
profiles/: <tag>_bench_lines.jsonl (every bench line), <tag>_{step,reset,vision}_ncu.txt (ncu --set
full metrics, hottest SASS and CUDA lines), <tag>_launches.txt (launch-list shares),
<tag>_sanitizer.txt, and the step kernel's per-launch DRAM traffic in ncu_step_summary.json."""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import make_profile_summary  # noqa: E402
import ncu_lines  # noqa: E402
import ncu_summary  # noqa: E402


def kernel_summary(rep):
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
    return "\n".join(lines) + "\n"


def main(run, tag):
    g = os.path.join(ROOT, "gpurun_out", run)
    P = os.path.join(ROOT, "profiles", tag)
    with open(P + "_bench_lines.jsonl", "w") as fh:
        for f in sorted(os.listdir(os.path.dirname(g))):
            if f.startswith(os.path.basename(g) + "_bench_") and f.endswith(".log"):
                last = [ln for ln in open(os.path.join(os.path.dirname(g), f)) if ln.startswith("{")]
                if last:
                    fh.write(json.dumps({"run": f[:-4], **json.loads(last[-1])}) + "\n")
    if os.path.exists(g + "_prof_step.ncu-rep"):
        make_profile_summary.main(tag, g + "_prof_step.ncu-rep", g + "_launches.csv",
                                  "cfg4-1M-envs-full-pipeline", 1 << 20)
    for k in ("reset", "vision"):
        if os.path.exists(g + f"_prof_{k}.ncu-rep"):
            open(P + f"_{k}_ncu.txt", "w").write(kernel_summary(g + f"_prof_{k}.ncu-rep"))
    if os.path.exists(g + "_prof_reset.ncu-rep"):   # the reset kernel's DRAM bytes per launch (config 5)
        full = ncu_summary.raw(g + "_prof_reset.ncu-rep")[0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb = float(full["dram__bytes_read.sum"][0]) * scale.get(full["dram__bytes_read.sum"][1], 1)
        wb = float(full["dram__bytes_write.sum"][0]) * scale.get(full["dram__bytes_write.sum"][1], 1)
        js_path = os.path.join(ROOT, "profiles", "ncu_step_summary.json")
        js = json.load(open(js_path)) if os.path.exists(js_path) else {}
        wi = float(full["smsp__inst_executed.sum"][0]) if "smsp__inst_executed.sum" in full else None
        js["cfg5-reset-kernel"] = {"tag": tag, "dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                                   "resets_per_launch": 104857, "warp_instructions": wi}
        json.dump(js, open(js_path, "w"), indent=1)
    out = []
    for t in ("memcheck", "racecheck", "synccheck", "initcheck"):
        f = g + f"_sanitize_{t}.log"
        if os.path.exists(f):
            txt = open(f).read()
            keep = [ln for ln in txt.splitlines() if re.search(r"SUMMARY|sanitize paths OK|Invalid|Race|Barrier", ln)]
            out.append(f"== {t}\n" + "\n".join(keep))
    if out:
        out.append("memcheck 'errors', if any, are leak reports: check their allocation frames (torch's caching "
                   "allocators vs libdr) in gpurun_out/" + run + "_sanitize_memcheck.log.")
        open(P + "_sanitizer.txt", "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
