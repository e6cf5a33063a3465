#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export DR_STEP_MODE=throughput
python scripts/dbg_dump.py full 511 200 16
RESET_T=99 python scripts/dbg_dump.py smooth_noreset 1023 200 16
python scripts/dbg_dump.py smooth_1000 1023 1000 16
