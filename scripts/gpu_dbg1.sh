#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
V=$PWD/paper_1906_11633_b200/variants/old.so
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "smoothing_and_substep and throughput" > gpurun_out/dbg_new.log 2>&1; tail -5 gpurun_out/dbg_new.log | cut -c1-300
DR_LIB=$V timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "smoothing_and_substep and throughput" > gpurun_out/dbg_old.log 2>&1; tail -5 gpurun_out/dbg_old.log | cut -c1-300
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/dbg_new_step -f python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
DR_LIB=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/dbg_old_step -f python bench.py --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/
