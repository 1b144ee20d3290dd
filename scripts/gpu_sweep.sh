set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python scripts/time_c4.py variants/prof.so > gpurun_out/sweep26.log 2>&1
cat gpurun_out/sweep26.log
