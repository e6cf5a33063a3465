#!/bin/bash
# HEAD check: smoke, every GPU test, and the bench lines (default, reset, vision, cfg2, cfg3).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/head
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv > ${O}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > ${O}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest_gpu.log
tail -3 ${O}_pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > ${O}_bench_default.log 2>&1; tail -1 ${O}_bench_default.log | cut -c1-300
for c in reset vision cfg2 cfg3; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-500} --warmup 20 --no-cpu-baseline > ${O}_bench_$c.log 2>&1
  tail -1 ${O}_bench_$c.log | cut -c1-300
done
echo done
