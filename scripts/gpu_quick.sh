#!/bin/bash
# GPU tests (all, or PYTEST_K) + small-config benches with CUDA graphs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-cfg2 cfg3}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-1000} --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
echo done
