#!/bin/bash
# Reset parity tests of the current build + A/B of variants/old.so vs variants/new.so on config 5.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "reset" > gpurun_out/abr_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/abr_pytest.log; tail -2 gpurun_out/abr_pytest.log
for rep in 1 2 3; do for v in old new; do
  DR_LIB=variants/$v.so timeout 300 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abr_${v}_r$rep.log 2>&1
  echo "reset $v r$rep: $(tail -1 gpurun_out/abr_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["split"]["reset_ms_avg"])')"
done; done
