#!/bin/bash
# Vision GPU tests (both augmentation modes) + bench --config vision for each mode, then one
# ncu --set full capture of the two-pass kernels.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vision.py -q -rf > gpurun_out/pytest_vision.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_vision.log
tail -3 gpurun_out/pytest_vision.log
for rep in 1 2; do
  for m in two_pass cluster; do
    DR_IMG_MODE=$m timeout 300 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/vision_${m}_r$rep.log 2>&1
    echo "vision $m r$rep: $(tail -1 gpurun_out/vision_${m}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d.get("roofline"), d["clocks"])')"
  done
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"image_noise|image_moments" -s 4 -c 2 -o gpurun_out/prof_vision2 -f \
      python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_vision2.log 2>&1
fi
echo done
