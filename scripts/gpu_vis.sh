#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_vision.py -m gpu -q -x > gpurun_out/vis_test.log 2>&1; echo "vision tests rc=$?"; tail -3 gpurun_out/vis_test.log | cut -c1-300
for r in 1 2; do for v in ${VARIANTS:-ilp1 ilp2 ilp4}; do
  echo "$v r$r: $(DR_LIB=variants/$v.so timeout 120 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 0 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3, d["clocks"]["sm_mhz"])')"
done; done
