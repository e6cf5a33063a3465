#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do for v in "$@"; do
  DR_LIB=variants/$v.so timeout 300 python bench.py --config vision --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step']*1e3, 2), 'us', d['value'])"
done; done
