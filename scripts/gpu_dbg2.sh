#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "smoothing_and_substep" > gpurun_out/dbg2_sub$i.log 2>&1; tail -3 gpurun_out/dbg2_sub$i.log | cut -c1-300
done
timeout 600 python -m pytest tests/test_gpu_edge_cases.py -m gpu -q -rA > gpurun_out/dbg2_edge.log 2>&1; tail -15 gpurun_out/dbg2_edge.log | cut -c1-400
NOTEST=1 CONFIGS="full1m reset" NCU="step_kernel" bash scripts/gpu_iter.sh
