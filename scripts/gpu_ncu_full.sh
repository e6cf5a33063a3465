#!/bin/bash
# ncu --set full of one kernel: KREGEX (step_kernel | reset_kernel | image_augment), CONFIG (bench --config), TAG
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-step_kernel} -s 3 -c 1 \
    -o gpurun_out/${TAG:-cur}_${KREGEX:-step_kernel} -f python bench.py --config ${CONFIG:-full1m} --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG:-cur}_ncu.log 2>&1
ls -la gpurun_out/${TAG:-cur}_${KREGEX:-step_kernel}.ncu-rep
