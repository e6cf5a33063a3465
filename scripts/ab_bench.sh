#!/bin/bash
# A/B: run bench.py (1M envs, full) for each variant library; one JSON line per variant and repeat.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
  for v in "$@"; do
    DR_LIB=variants/$v.so timeout 300 python bench.py --steps ${STEPS:-1000} --warmup 20 --no-cpu-baseline --e2e-steps 0 ${EXTRA} > gpurun_out/ab_${v}_r$rep.log 2>&1
  done
done
echo done
