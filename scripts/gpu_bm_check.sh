cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for mode in throughput latency; do
  for v in oldbm newbm; do DR_STEP_MODE=$mode DR_LIB=variants/$v.so python scripts/bitident.py /tmp/bi_${v}_$mode.npz || echo "dump failed $v"; done
  echo "$mode: $(python scripts/bitident.py --compare /tmp/bi_oldbm_$mode.npz /tmp/bi_newbm_$mode.npz)"
done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash scripts/ab_reset_variants.sh oldbm newbm
