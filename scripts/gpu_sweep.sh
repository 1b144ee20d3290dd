set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PREROLL=200
timeout 200 python scripts/time_c4.py > gpurun_out/sweep30.log 2>&1
for v in noflat flat16 flat8; do timeout 200 python scripts/time_c4.py variants/$v.so; done >> gpurun_out/sweep30.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py tests/test_gpu_capacity.py -x -q -m gpu -k "not full_run" > gpurun_out/gputests30.log 2>&1
tail -3 gpurun_out/gputests30.log
cat gpurun_out/sweep30.log
