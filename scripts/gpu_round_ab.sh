#!/bin/bash
# GPU tests + A/B benches: reset kernels (VERSIONS), the default 1M step bench (REPS times) and
# the vision bench.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for v in ${VERSIONS:-6 3}; do
    DR_RESET=$v timeout 300 python bench.py --config reset --steps 200 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/reset_v${v}_r$rep.log 2>&1
    echo "reset v$v r$rep: $(tail -1 gpurun_out/reset_v${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["clocks"])')"
  done
done
for rep in $(seq 1 ${REPS:-2}); do
  timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/step_r$rep.log 2>&1
  echo "step r$rep: $(tail -1 gpurun_out/step_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"])')"
done
timeout 300 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/vision.log 2>&1
echo "vision: $(tail -1 gpurun_out/vision.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"])')"
echo done
