#!/bin/bash
# Vision check at HEAD: vision GPU tests, bench --config vision (3 runs), ncu --set full of the
# augmentation kernel.  Output gpurun_out/${TAG}_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/${TAG:-vc}
timeout 600 python -m pytest tests/test_gpu_vision.py tests/test_gpu_examples.py -q > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
for r in 1 2 3; do timeout 300 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline > ${O}_bench_r$r.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:image_augment -s 3 -c 1 -o ${O}_prof_vision -f \
    python bench.py --config vision --profile --steps 6 --warmup 3 --no-cpu-baseline > ${O}_ncu_vision.log 2>&1
tail -n 2 ${O}_pytest.log
for r in 1 2 3; do tail -n 1 ${O}_bench_r$r.log | cut -c1-200; done
