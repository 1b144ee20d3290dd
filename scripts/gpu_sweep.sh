set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python -m pytest tests/test_gpu_merge.py tests/test_gpu_capacity.py tests/test_gpu_partition.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gputests27.log 2>&1
tail -30 gpurun_out/gputests27.log
