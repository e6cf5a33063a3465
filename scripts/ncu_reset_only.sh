#!/bin/bash
# ncu --set full of the reset kernels (config 5) of the current build (TAG names the report).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reset_ -s 6 -c 2 -o gpurun_out/prof_reset_$TAG -f \
    python bench.py --config reset --profile --steps 6 --warmup 3 --no-cpu-baseline ${EXTRA} > gpurun_out/ncu_reset_$TAG.log 2>&1
echo done
