cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
DR_LIB=variants/dbg.so timeout 300 python scripts/reset_check_1m.py /tmp/rc_dbg.npz > gpurun_out/rc_dbg.log 2>&1
for v in old new; do DR_LIB=variants/$v.so timeout 300 python scripts/reset_check_1m.py /tmp/rc_$v.npz > gpurun_out/rc_$v.log 2>&1; done
python scripts/reset_check_1m.py --compare /tmp/rc_old.npz /tmp/rc_new.npz
tail -n 3 gpurun_out/rc_old.log gpurun_out/rc_new.log
grep -c "reset n=" gpurun_out/rc_dbg.log; grep "reset n=" gpurun_out/rc_dbg.log | head -8; tail -2 gpurun_out/rc_dbg.log
