#!/bin/bash
# Prefetch-policy sweep of the step kernel at 1M envs (full pipeline).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for pf in 0 1 2; do
  DR_PREFETCH=$pf timeout 300 python bench.py --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline --e2e-steps 0 ${EXTRA} > gpurun_out/pf$pf.log 2>&1
done
echo done
