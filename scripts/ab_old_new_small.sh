#!/bin/bash
# A/B of variants/old.so vs variants/new.so on the small configs (cfg2 latency kernel, cfg3) and 1M,
# after the GPU parity tests of the current build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log; tail -2 gpurun_out/ab_pytest.log
for rep in 1 2 3; do for v in old new; do
  for c in ${CONFIGS:-cfg2 cfg3 full1m}; do
    steps=2000; [ $c = cfg2 ] && steps=5000
    DR_LIB=variants/$v.so timeout 300 python bench.py --config $c --steps $steps --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abs_${c}_${v}_r$rep.log 2>&1
    echo "$c $v r$rep: $(tail -1 gpurun_out/abs_${c}_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, "us", d["value"], d["clocks"]["sm_mhz"])')"
  done
done; done
