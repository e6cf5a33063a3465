#!/bin/bash
# Step-kernel occupancy A/B (DR_STEP_MIN_CTAS variants from build_variants.sh): bit identity
# against base (scripts/bitident.py), then three alternating default-bench runs per variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="${VARIANTS:-base s5 s6}"
for v in $V; do DR_LIB=variants/$v.so timeout 300 python scripts/bitident.py /tmp/sb_$v.npz > gpurun_out/socc_bitident_$v.log 2>&1; done
for v in $V; do python scripts/bitident.py --compare /tmp/sb_base.npz /tmp/sb_$v.npz >> gpurun_out/socc_bitident.txt 2>&1; echo "$v rc=$?" >> gpurun_out/socc_bitident.txt; done
CONFIG=${CONFIG:-full1m} STEPS=${STEPS:-2000} VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/socc_ab.txt 2>&1
cat gpurun_out/socc_bitident.txt gpurun_out/socc_ab.txt
