#!/bin/bash
# Round-2 opening measurement: smoke, default bench, strong-scaling proxies (1M/8, 1M/4 per GPU,
# graph-captured), reset and vision configs.  gpurun_out/r2base_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2base
nvidia-smi > ${O}_nvidia-smi.txt 2>&1
lscpu > ${O}_lscpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout 900 python bench.py > ${O}_bench_default.log 2>&1
for n in 131072 262144 524288; do
  timeout 300 python bench.py --n-env $n --graph 100 --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 3 > ${O}_bench_n$n.log 2>&1
done
timeout 600 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline > ${O}_bench_reset.log 2>&1
timeout 600 python bench.py --config vision --steps 500 --warmup 20 --no-cpu-baseline > ${O}_bench_vision.log 2>&1
echo done
