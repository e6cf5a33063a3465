#!/bin/bash
# Bench lines of every config (no CPU baseline), summarised; gpurun_out/q_*.log.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in full1m reset cfg3 cfg2 vision; do
  case $c in cfg2) st=5000;; cfg3) st=2000;; reset) st=300;; vision) st=500;; *) st=2000;; esac
  timeout 600 python bench.py --config $c --steps $st --warmup 20 --no-cpu-baseline > gpurun_out/q_$c.log 2>&1
  tail -1 gpurun_out/q_$c.log | python -c '
import json,sys
d=json.loads(sys.stdin.read()); r=d["roofline"]
print(sys.argv[1], "%.4g" % d["value"], d["unit"], "ms %.5f" % d["ms_per_step"], "frac %.3f" % r["frac"], "e2e %.3g" % (d.get("e2e") or {}).get("value", 0), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"], "split", json.dumps(r.get("split", {}).get("reset_ms_avg")))' $c
done
