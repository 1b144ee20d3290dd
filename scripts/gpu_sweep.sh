cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 bash scripts/sanitize.sh
export PREROLL=200
timeout 200 python scripts/time_c4.py > gpurun_out/sweep35.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputests35.log 2>&1
tail -3 gpurun_out/gputests35.log
cat gpurun_out/sweep35.log
