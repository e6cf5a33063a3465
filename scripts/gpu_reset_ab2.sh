#!/bin/bash
# Reset rework check: GPU tests (PYTEST_K), bit identity old vs new (scripts/bitident.py), config-5
# A/B of VARIANTS (variants/<v>.so; default "old new"), three alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/rab
timeout 1200 python -m pytest tests -m gpu -q -x -rf ${PYTEST_K:+-k "$PYTEST_K"} > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log; tail -3 ${O}_pytest.log
for v in old new; do DR_LIB=variants/$v.so timeout 300 python scripts/bitident.py gpurun_out/bi_$v.npz > ${O}_bi_$v.log 2>&1; done
python scripts/bitident.py --compare gpurun_out/bi_old.npz gpurun_out/bi_new.npz 2>&1 | tail -3
for rep in 1 2 3; do for v in ${VARIANTS:-old new}; do
  DR_LIB=variants/$v.so timeout 300 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 > ${O}_${v}_r$rep.log 2>&1
  echo "reset $v r$rep: $(tail -1 ${O}_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["split"]["reset_ms_avg"])')"
done; done
echo done
