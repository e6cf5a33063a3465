#!/bin/bash
# Readiness-poll back-off A/B (DR_POLL_NS variants): cfg2 and cfg3, three alternating runs each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="${VARIANTS:-base ns0 ns16 ns256}"
CONFIG=cfg2 STEPS=5000 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/poll_cfg2.txt 2>&1
CONFIG=cfg3 STEPS=2000 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/poll_cfg3.txt 2>&1
cat gpurun_out/poll_cfg2.txt gpurun_out/poll_cfg3.txt
