#!/bin/bash
# Full default bench line + the other configs + reset-kernel ncu, into gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_default.log 2>&1
for c in cfg2 cfg3 reset; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
if [ -n "$NCU_RESET" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:reset_kernel -s 4 -c 1 -o gpurun_out/prof_reset -f \
      python bench.py --config reset --profile --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_reset.log 2>&1
fi
echo done
