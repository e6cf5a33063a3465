#!/bin/bash
# Per-GPU throughput of the full pipeline across env counts (one GPU; CUDA graphs below 200 MB per
# step as in bench.py): the HBM-bound rate should hold from the strong-split shards to 16M envs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for n in 131072 262144 524288 1048576 2097152 4194304 8388608 16777216; do
  steps=$(( n >= 4194304 ? 20 : 200 ))
  echo "n=$n $(timeout 600 python bench.py --n-env $n --steps $steps --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done
