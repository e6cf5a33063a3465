#!/bin/bash
# A/B of variant libraries (args) on config 5 (reset + step), three alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2 3; do for v in "$@"; do
  DR_LIB=variants/$v.so timeout 300 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abrv_${v}_r$rep.log 2>&1
  echo "reset $v r$rep: $(tail -1 gpurun_out/abrv_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["split"]["reset_ms_avg"])')"
done; done
