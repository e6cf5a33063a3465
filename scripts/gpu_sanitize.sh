#!/bin/bash
# compute-sanitizer over every libdr kernel path (scripts/sanitize_paths.py): memcheck, racecheck,
# synccheck, initcheck.  Output in gpurun_out/sanitize_<tool>.log.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --kernel-name kns=_ZN2dr \
      python scripts/sanitize_paths.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize paths OK' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
echo done
