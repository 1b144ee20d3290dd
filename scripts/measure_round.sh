#!/bin/bash
# All measurement artefacts of a round, on one B200 (run under gpurun):
#   bench lines (C4 2M, 8M, max pressure, oracle reference arm, batched),
#   ncu --set full of one k_step launch, and the cold launch list of bench.py.
# Outputs land in gpurun_out/; copy the summaries into profiles/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python bench.py > gpurun_out/bench.log 2>&1
python bench.py --scale 4 --steps 50 --no-cpu > gpurun_out/bench_8m.log 2>&1
python bench.py --policy maxpressure --no-cpu > gpurun_out/bench_mp.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python scripts/bench_batched.py > gpurun_out/bench_batched.log 2>&1
python scripts/bench_transport.py 8 > gpurun_out/transport.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 20 -c 1 \
    -o gpurun_out/prof_kstep -f python scripts/time_c4.py > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_kstep.ncu-rep --page source --csv > gpurun_out/kstep_source.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
tail -n 2 gpurun_out/bench*.log
