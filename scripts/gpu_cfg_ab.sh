#!/bin/bash
# A/B of VARIANTS (variants/<v>.so) on bench CONFIG (default cfg2), three alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for v in ${VARIANTS:-base new}; do
  echo "${CONFIG:-cfg2} $v r$rep: $(DR_LIB=variants/$v.so timeout 300 python bench.py --config ${CONFIG:-cfg2} --steps ${STEPS:-3000} --warmup 20 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1000, "us", d["value"])')"
done; done
