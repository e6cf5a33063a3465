#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
O=gpurun_out/r2b
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -rA > ${O}_multirank.log 2>&1; echo "multirank rc=$?"; grep -E "PASSED|FAILED|passed|failed" ${O}_multirank.log | tail -8
timeout 600 python bench.py > ${O}_bench_default.log 2>&1; tail -1 ${O}_bench_default.log
NOTEST=1 CONFIGS="n131k n262k reset cfg3" bash scripts/gpu_iter.sh
