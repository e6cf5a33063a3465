#!/bin/bash
# Vision register-cap A/B (DR_IMG_MINB / DR_IMG_PRE variants from build_variants.sh): bit identity
# against base, then three alternating bench --config vision runs per variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="${VARIANTS:-base p1 minb8p1 minb9 minb9p1 minb10p1}"
for v in $V; do DR_LIB=variants/$v.so timeout 300 python scripts/vision_bitident.py /tmp/vb_$v.npz > gpurun_out/vrc_bitident_$v.log 2>&1; done
for v in $V; do python scripts/vision_bitident.py --compare /tmp/vb_base.npz /tmp/vb_$v.npz >> gpurun_out/vrc_bitident.txt 2>&1; echo "$v rc=$?" >> gpurun_out/vrc_bitident.txt; done
CONFIG=vision STEPS=500 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/vrc_ab.txt 2>&1
cat gpurun_out/vrc_bitident.txt gpurun_out/vrc_ab.txt
