#!/bin/bash
# Reset-kernel A/B (variant libraries) + reset parity tests on the in-tree build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "reset or resume or edge or chain" > gpurun_out/rab_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/rab_pytest.log)"
bash scripts/ab_reset_variants.sh "$@"
