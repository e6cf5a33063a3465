#!/bin/bash
# Early-trigger A/B (DR_RESET_EARLY_TRIGGER / DR_STEP_EARLY_TRIGGER variants): bit identity, then
# config 5 (reset + step), the default 1M and config 3, three alternating runs each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="${VARIANTS:-base rt st rtst}"
for v in $V; do DR_LIB=variants/$v.so timeout 300 python scripts/bitident.py /tmp/tb_$v.npz > gpurun_out/trig_bitident_$v.log 2>&1; done
for v in $V; do python scripts/bitident.py --compare /tmp/tb_base.npz /tmp/tb_$v.npz >> gpurun_out/trig_bitident.txt 2>&1; echo "$v rc=$?" >> gpurun_out/trig_bitident.txt; done
CONFIG=reset STEPS=300 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/trig_reset.txt 2>&1
CONFIG=full1m STEPS=2000 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/trig_full1m.txt 2>&1
CONFIG=cfg3 STEPS=2000 VARIANTS="$V" bash scripts/gpu_cfg_ab.sh > gpurun_out/trig_cfg3.txt 2>&1
cat gpurun_out/trig_bitident.txt gpurun_out/trig_reset.txt gpurun_out/trig_full1m.txt gpurun_out/trig_cfg3.txt
