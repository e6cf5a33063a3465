cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do for x in 1 2 3.46 4 8; do
  echo "x=$x r$r: $(DR_RESET_GRID_X=$x DR_LIB=variants/new.so timeout 300 python bench.py --config reset --steps 300 --warmup 10 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["split"]["reset_ms_avg"])')"
done; done
