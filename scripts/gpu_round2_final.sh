#!/bin/bash
# Round-2 evidence in one call: smoke, GPU tests, every bench line (default with cpu_baseline and
# e2e; cfg2/cfg3/reset/vision; the reference arm), the PCIe probe, the ncu launch list of the
# default bench and ncu --set full captures of the step, reset and image kernels.  gpurun_out/final_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/${TAG:-r7}
nvidia-smi > ${O}_nvidia-smi.txt 2>&1
lscpu > ${O}_lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA > ${O}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest_gpu.log
timeout 900 python bench.py > ${O}_bench_default.log 2>&1
timeout 600 python bench.py --config cfg2 --steps 5000 --warmup 20 --no-cpu-baseline > ${O}_bench_cfg2.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 2000 --warmup 20 --no-cpu-baseline > ${O}_bench_cfg3.log 2>&1
timeout 600 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline > ${O}_bench_reset.log 2>&1
timeout 600 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline > ${O}_bench_vision.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_reference.log 2>&1
for n in 524288 262144 131072; do
  timeout 600 python bench.py --n-env $n --steps 4000 --warmup 20 --no-cpu-baseline > ${O}_bench_n$n.log 2>&1
done
timeout 300 python scripts/pcie_probe.py > ${O}_pcie.log 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/bw_ceiling scripts/bw_ceiling.cu && \
  timeout 300 /tmp/bw_ceiling 1.0 8 20 1 > ${O}_bw_ceiling_1gb_pdl.txt 2>&1 && \
  timeout 300 /tmp/bw_ceiling 0.115 8 200 1 > ${O}_bw_ceiling_115mb_pdl.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"step_kernel|reset_kernel|augment|scene|pose|image_" -c 40 --csv --log-file ${O}_launches.csv \
    python bench.py --profile --steps 30 --warmup 5 --no-cpu-baseline > ${O}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o ${O}_prof_step -f \
    python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > ${O}_ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:reset_kernel -s 3 -c 1 -o ${O}_prof_reset -f \
    python bench.py --config reset --profile --steps 6 --warmup 3 --no-cpu-baseline > ${O}_ncu_reset.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_augment -s 3 -c 1 -o ${O}_prof_vision -f \
    python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline > ${O}_ncu_vision.log 2>&1
# compute-sanitizer is closed on this GPU pool since the round-2 v2 run (profiles/README.md); the
# last sanitizer pass is profiles/round2_v1_sanitizer.txt.  SANITIZE=1 runs it where it is allowed.
if [ "${SANITIZE:-0}" = 1 ]; then
  bash scripts/gpu_sanitize.sh > ${O}_sanitize.log 2>&1
  for t in memcheck racecheck synccheck initcheck; do cp gpurun_out/sanitize_$t.log ${O}_sanitize_$t.log 2>/dev/null; done
fi
echo done
