#!/bin/bash
# dr_reset alone (scripts/reset_probe.py) for VARIANTS, three alternating runs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for v in ${VARIANTS:-old new}; do
  echo "$v r$rep: $(DR_LIB=variants/$v.so timeout 120 python scripts/reset_probe.py 2>&1 | tail -1)"
done; done
