#!/bin/bash
# All measurement artefacts of a round, on one B200 (run under gpurun):
#   bench lines (C4 2M, 8M, max pressure, oracle reference arm, batched),
#   ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
tail -n 2 gpurun_out/bench*.log
