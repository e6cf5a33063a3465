#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
DR_STEP_MODE=throughput RESET_T=9 timeout 600 compute-sanitizer --tool racecheck --kernel-name kns=step_kernel python scripts/dbg_dump.py san 1023 200 13 > gpurun_out/san_racecheck.log 2>&1
echo "racecheck: $(grep -E 'RACECHECK SUMMARY|dumped' gpurun_out/san_racecheck.log | tr '\n' ' ')"
NCU="step_kernel" bash scripts/gpu_iter.sh
