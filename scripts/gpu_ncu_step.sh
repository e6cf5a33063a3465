#!/bin/bash
# ncu --set full of the step kernel (default bench workload) -> gpurun_out/${TAG:-cur}_step.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/${TAG:-cur}_step -f python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/${TAG:-cur}_step.ncu-rep
