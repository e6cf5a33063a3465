#!/bin/bash
# Vision A/B: GPU vision tests, bench --config vision per forced cluster size (DR_IMG_K; 0 = the
# balanced default), optional ncu --set full of image_augment_kernel.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_vision.py -q > gpurun_out/pytest_vision.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_vision.log
for rep in 1 2; do
  for k in ${KS:-0 4}; do
    if [ "$k" = 0 ]; then unset DR_IMG_K; else export DR_IMG_K=$k; fi
    timeout 300 python bench.py --config vision --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/vision_k${k}_r$rep.log 2>&1
  done
done
unset DR_IMG_K
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_augment -s 4 -c 1 -o gpurun_out/prof_vision -f \
      python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_vision.log 2>&1
fi
echo done
