#!/bin/bash
# GPU tests (PDL on, the default) + A/B of DR_PDL=1/0 on every DR config.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  for c in cfg2 cfg3 full1m reset; do
    for pdl in 1 0; do
      steps=2000; [ $c = cfg2 ] && steps=5000; [ $c = reset ] && steps=300
      DR_PDL=$pdl timeout 300 python bench.py --config $c --steps $steps --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pdl_${c}_${pdl}_r$rep.log 2>&1
      echo "$c pdl=$pdl r$rep: $(tail -1 gpurun_out/pdl_${c}_${pdl}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
    done
  done
done
echo done
