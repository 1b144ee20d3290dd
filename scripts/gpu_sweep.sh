set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python scripts/time_c4.py > gpurun_out/sweep6.log 2>&1
for v in prof cw8 cw10; do timeout 300 python scripts/time_c4.py variants/$v.so; done >> gpurun_out/sweep6.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "one_step or exact_mode" > gpurun_out/parity6.log 2>&1
tail -3 gpurun_out/parity6.log
cat gpurun_out/sweep6.log
