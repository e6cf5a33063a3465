#!/bin/bash
# HBM ceilings of the libdr read/write mixes (scripts/bw_ceiling.cu): 1 GB per launch (ring of 2)
# and the vision batch's size (115 MB per launch, ring of 4, as bench --config vision); then both
# with programmatic dependent launch and a ring of 8 (several small-grid launches can be resident at
# once: with a ring of 2 they shared input buffers through L2 and read > 8 TB/s).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/${TAG:-bwc}
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/bw_ceiling scripts/bw_ceiling.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > ${O}_clocks_before.txt
timeout 300 /tmp/bw_ceiling 1.0 2 20 > ${O}_1gb.txt 2>&1
timeout 300 /tmp/bw_ceiling 0.115 4 200 > ${O}_115mb.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > ${O}_clocks_after.txt
grep '^{' ${O}_1gb.txt ${O}_115mb.txt
timeout 300 /tmp/bw_ceiling 0.115 8 200 1 > ${O}_115mb_pdl.txt 2>&1
timeout 300 /tmp/bw_ceiling 1.0 8 20 1 > ${O}_1gb_pdl.txt 2>&1
grep '^{' ${O}_115mb_pdl.txt ${O}_1gb_pdl.txt
