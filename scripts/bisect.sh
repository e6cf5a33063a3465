#!/bin/bash
# Bisect the small-n parity failures: pipe variants, the previous library build, and sanitizers.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
K='test_ragged_sizes or test_layer_subsets or test_config1'
for cfg in "p0::0" "p1::1" "p2::2" "prev:variants/prev.so:2" "prev0:variants/prev.so:0"; do
  name=${cfg%%:*}; rest=${cfg#*:}; lib=${rest%%:*}; pipe=${rest#*:}
  if [ -n "$lib" ]; then export DR_LIB=$lib; else unset DR_LIB; fi
  DR_PIPE=$pipe timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$K" > gpurun_out/bisect_$name.log 2>&1
  tail -3 gpurun_out/bisect_$name.log
done
unset DR_LIB
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "test_ragged_sizes and 1]" > gpurun_out/san_$tool.log 2>&1
  tail -30 gpurun_out/san_$tool.log | head -40
done
