set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python scripts/time_c4.py > gpurun_out/sweep24.log 2>&1
timeout 120 python scripts/time_c4.py variants/prof.so >> gpurun_out/sweep24.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests24.log 2>&1
tail -3 gpurun_out/gputests24.log
cat gpurun_out/sweep24.log
