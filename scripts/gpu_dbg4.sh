#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export DR_STEP_MODE=throughput RESET_T=99
for tool in racecheck synccheck initcheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --kernel-name kns=step_kernel python scripts/dbg_dump.py san 1023 200 13 > gpurun_out/san_$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|dumped' gpurun_out/san_$tool.log | tr '\n' ' ')"
done
