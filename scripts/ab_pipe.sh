#!/bin/bash
# A/B over (library variant, DR_PIPE) pairs: "lib:pipe" arguments; one bench JSON per pair.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "$@"; do
  lib=${v%%:*}; pipe=${v#*:}
  DR_LIB=variants/$lib.so DR_PIPE=$pipe timeout 300 python bench.py --steps ${STEPS:-1000} --warmup 20 --no-cpu-baseline --e2e-steps 0 ${EXTRA} > gpurun_out/ab_${lib}_p${pipe}.log 2>&1
done
echo done
