set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1500 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_ipc.py tests/test_gpu_parity.py -x -q -m gpu -k "boundary or device or allocator or ipc or full_run" > gpurun_out/gputests28.log 2>&1
tail -30 gpurun_out/gputests28.log
