#!/bin/bash
# Vision A/B over (variant library, forced cluster size K) pairs "variant:K" (K = 0: the library's own
# choice), three alternating runs; prints us per 192-image batch.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2 3; do for vk in "$@"; do
  v=${vk%%:*}; k=${vk#*:}
  if [ "$k" = "0" ]; then envk=""; else envk="DR_IMG_K=$k"; fi
  echo "$vk r$r: $(env $envk DR_LIB=variants/$v.so timeout 300 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3, 3))' 2>&1 | tail -1)"
done; done
