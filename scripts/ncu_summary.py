#!/usr/bin/env python
"""Summarise an ncu report (raw metrics + hottest SASS lines) as text/JSON for profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


def hot_sass(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            data.append((int(r[iss]), r[ia], r[isrc], int(r[ie] or 0)))
        except ValueError:
            continue
    tot = sum(d[0] for d in data) or 1
    lines = [f"total stall samples {tot}, SASS instructions {len(data)}, executed {sum(d[3] for d in data)}"]
    for s, a, src, e in sorted(data, reverse=True)[:top]:
        lines.append(f"{s:7d} {100 * s / tot:5.1f}%  {src[:100]}")
    # opcode histogram of executed instructions
    hist = {}
    for s, a, src, e in data:
        op = src.split()[0] if src.split() else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        hist[op] = hist.get(op, 0) + e
    tot_e = sum(hist.values()) or 1
    lines.append("executed-instruction mix: " + ", ".join(f"{k} {100 * v / tot_e:.1f}%" for k, v in
                                                       sorted(hist.items(), key=lambda x: -x[1])[:24]))
    return lines


if __name__ == "__main__":
    rep = sys.argv[1]
    for d in raw(rep):
        print(d.pop("kernel")[:120])
        for k, (v, u) in d.items():
            print(f"  {k:80s} {v} {u}")
    if "--sass" in sys.argv:
        print("\n".join(hot_sass(rep)))
