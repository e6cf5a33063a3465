#!/bin/bash
# Bit identity of variants/old.so and variants/new.so on config 5's reset pattern at 1M envs
# (scripts/reset_check_1m.py; the dumps stay on the box's /tmp, only the logs come back).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in old new; do DR_LIB=variants/$v.so timeout 300 python scripts/reset_check_1m.py /tmp/rc_$v.npz > gpurun_out/rc_$v.log 2>&1; done
python scripts/reset_check_1m.py --compare /tmp/rc_old.npz /tmp/rc_new.npz
tail -n 3 gpurun_out/rc_old.log gpurun_out/rc_new.log
