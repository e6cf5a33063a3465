#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_chain.py -m gpu -q -x > gpurun_out/chain_test.log 2>&1; echo "chain test rc=$?"; tail -3 gpurun_out/chain_test.log | cut -c1-300
VAR=DR_CHAIN VALUES=0,1 SIZES="131072 262144 65536" bash scripts/ab_env_small.sh
for v in 0 1; do DR_CHAIN=$v timeout 120 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/chain_full_$v.log 2>&1; echo "1M DR_CHAIN=$v $(tail -1 gpurun_out/chain_full_$v.log | cut -c1-200)"; done
