cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log; tail -2 gpurun_out/ab_pytest.log
for rep in 1 2 3; do for v in old new; do
  DR_LIB=variants/$v.so timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_${v}_r$rep.log 2>&1
  echo "1M $v r$rep: $(tail -1 gpurun_out/ab_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
  DR_LIB=variants/$v.so timeout 300 python bench.py --config cfg3 --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab3_${v}_r$rep.log 2>&1
  echo "cfg3 $v r$rep: $(tail -1 gpurun_out/ab3_${v}_r$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done; done
