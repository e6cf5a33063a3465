#!/bin/bash
# A/B of an environment knob (VAR=v1,v2,...) on the n131k / n262k / cfg3 configs, two alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
IFS=',' read -ra VALS <<< "$VALUES"
for rep in 1 2; do for v in "${VALS[@]}"; do for n in ${SIZES:-131072 262144}; do
  env $VAR=$v timeout 120 python bench.py --n-env $n --graph 100 --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abe_${v}_$n.log 2>&1
  echo "$VAR=$v n=$n r$rep: $(tail -1 gpurun_out/abe_${v}_$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.4g" % d["value"], "%.5f" % d["ms_per_step"], d["clocks"]["sm_mhz"])')"
done; done; done
