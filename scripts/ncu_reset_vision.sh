#!/bin/bash
# ncu --set full captures (with source) of the reset kernel (config 5) and the image-augment kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-rv}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reset_kernel -s 3 -c 1 -o gpurun_out/prof_reset_$TAG -f \
    python bench.py --config reset --profile --steps 6 --warmup 3 --no-cpu-baseline ${EXTRA} > gpurun_out/ncu_reset_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_augment -s 3 -c 1 -o gpurun_out/prof_vision_$TAG -f \
    python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline ${EXTRA} > gpurun_out/ncu_vision_$TAG.log 2>&1
echo done
