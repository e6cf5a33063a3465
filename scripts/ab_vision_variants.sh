#!/bin/bash
# A/B of variant libraries (args) on the vision config, three alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2 3; do for v in "$@"; do
  echo "$v r$r: $(DR_LIB=variants/$v.so python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 0 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"]*1e3)')"
done; done
