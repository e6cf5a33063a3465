#!/bin/bash
# Reset-kernel A/B: GPU tests with the default kernel, bench --config reset for each DR_RESET
# version, one ncu --set full capture of the default reset kernel.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for v in ${VERSIONS:-5 3}; do
    DR_RESET=$v timeout 300 python bench.py --config reset --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/reset_v${v}_r$rep.log 2>&1
  done
done
if [ -n "$NCU_RESET" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:reset_kernel -s 4 -c 1 -o gpurun_out/prof_reset -f \
      python bench.py --config reset --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_reset.log 2>&1
fi
echo done
