#!/bin/bash
# A/B of variant libraries (args) on config 2 (latency kernel) and config 3; no tests (probes).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in 1 2; do for v in "$@"; do for c in ${CONFIGS:-cfg2 cfg3}; do
  steps=2000; [ $c = cfg2 ] && steps=5000
  DR_LIB=variants/$v.so timeout 300 python bench.py --config $c --steps $steps --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abp_${c}_${v}_r$rep.log 2>&1
  echo "$c $v r$rep: $(tail -1 gpurun_out/abp_${c}_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, "us")')"
done; done; done
