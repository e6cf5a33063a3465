#!/bin/bash
# ncu captures of the step kernel at 1M envs (full pipeline): launch list of our kernels + one --set full.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-step}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"step_kernel|reset_kernel|augment|scene|pose" -c 30 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --profile --steps 20 --warmup 5 --no-cpu-baseline ${EXTRA} > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_$TAG -f \
    python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline ${EXTRA} > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
