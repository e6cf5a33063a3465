#!/bin/bash
# A/B over environment settings of the default build: "name:VAR=value[,VAR=value]" arguments.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for rep in $(seq 1 ${REPS:-1}); do
  for v in "$@"; do
    name=${v%%:*}; envs=${v#*:}
    env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --steps ${STEPS:-1000} --warmup 20 --no-cpu-baseline --e2e-steps 0 ${EXTRA} > gpurun_out/ab_${name}_r$rep.log 2>&1
  done
done
echo done
