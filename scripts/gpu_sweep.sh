set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 120 python scripts/time_c4.py > gpurun_out/sweep18.log 2>&1
for v in free prof cw10 cw14; do timeout 120 python scripts/time_c4.py variants/$v.so; done >> gpurun_out/sweep18.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests18.log 2>&1
tail -3 gpurun_out/gputests18.log
cat gpurun_out/sweep18.log
