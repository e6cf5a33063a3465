#!/bin/bash
# A/B of library variants on the small configs (cfg2, cfg3): "lib:mode" arguments.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "$@"; do
  lib=${v%%:*}; mode=${v#*:}
  for c in cfg2 cfg3; do
    DR_LIB=variants/$lib.so DR_STEP_MODE=$mode timeout 300 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline --e2e-steps 0 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $mode $c', round(d['ms_per_step']*1e3, 2), 'us')"
  done
done
