#!/bin/bash
# Iteration check: GPU tests (all, or PYTEST_K), then the bench configs in CONFIGS (default: full1m
# reset), then optional ncu DRAM-byte captures of the kernels named in NCU (regex list, e.g.
# "step_kernel reset_kernel").  Output: gpurun_out/it_*.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/it
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -rf ${PYTEST_K:+-k "$PYTEST_K"} > ${O}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest_gpu.log
  tail -4 ${O}_pytest_gpu.log
fi
for c in ${CONFIGS:-full1m reset}; do
  case $c in
    full1m) args="--steps 2000 --warmup 20";;
    reset) args="--config reset --steps 300 --warmup 10";;
    cfg2) args="--config cfg2 --steps 5000 --warmup 20";;
    cfg3) args="--config cfg3 --steps 2000 --warmup 20";;
    vision) args="--config vision --steps 500 --warmup 20";;
    n131k) args="--n-env 131072 --graph 100 --steps 2000 --warmup 20";;
    n262k) args="--n-env 262144 --graph 100 --steps 2000 --warmup 20";;
  esac
  timeout 300 python bench.py $args --no-cpu-baseline --e2e-steps 3 > ${O}_bench_$c.log 2>&1
  tail -1 ${O}_bench_$c.log | python -c '
import json,sys
try:
    d=json.loads(sys.stdin.read()); r=d["roofline"]
    print("'$c'", "value %.4g" % d["value"], "ms %.5f" % d["ms_per_step"], "frac %.3f" % r["frac"], r.get("split",""), "clk", d.get("clocks",{}).get("sm_mhz"))
except Exception as e: print("'$c' parse error", e)'
done
for k in $NCU; do
  case $k in
    reset_kernel) args="--config reset";;
    image_augment) args="--config vision";;
    *) args="";;
  esac
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,sm__cycles_active.avg --clock-control none \
      -k regex:$k -s 3 -c 3 --csv --log-file ${O}_ncu_$k.csv python bench.py $args --profile --steps 6 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python scripts/ncu_metrics.py ${O}_ncu_$k.csv || tail -5 ${O}_ncu_$k.csv
done
echo done
