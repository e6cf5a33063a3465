#!/bin/bash
# Vision bench line + ncu launch list and one full capture of image_augment_kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python bench.py --config vision --steps ${STEPS:-200} --warmup 10 > gpurun_out/bench_vision.log 2>&1
tail -1 gpurun_out/bench_vision.log | cut -c1-600
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"augment|scene" -c 20 --csv --log-file gpurun_out/launches_vision.csv \
      python bench.py --config vision --profile --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_vision.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_augment -s 4 -c 1 -o gpurun_out/prof_vision -f \
      python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_vision.log 2>&1
fi
echo done
