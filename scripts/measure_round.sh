#!/bin/bash
# All measurement artefacts of a round, on one B200 (run under gpurun):
#   ncu --set full captures of one k_step launch after the bench's 200-step
#   pre-roll (C4 2M and the 8M instance), summarised into profiles/ first so
#   the bench lines carry this build's DRAM traffic / issue fraction; bench
#   lines (C4 2M, 8M, max pressure, oracle reference arm, batched); the floor /
#   peak numbers; the cold launch list of bench.py.  ROUND=r02 names the files.
set -x
R=${ROUND:-r02}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PREROLL=200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 210 -c 1 \
    -o gpurun_out/prof_kstep -f python scripts/time_c4.py > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_kstep.ncu-rep --page source --csv --print-source sass > gpurun_out/kstep_source.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof_kstep.ncu-rep profiles/${R}_kstep_ncu_full.txt \
    profiles/ncu_kstep_traffic.json > /dev/null
SCALE=4 timeout 900 ncu --set full --clock-control none -k regex:k_step -s 210 -c 1 \
    -o gpurun_out/prof_kstep_8m -f python scripts/time_c4.py > gpurun_out/ncu_full_8m.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_kstep_8m.ncu-rep profiles/${R}_kstep_ncu_full_8m.txt \
    profiles/ncu_kstep_traffic_8m.json 8000000 > /dev/null
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --scale 4 --steps 50 --no-cpu > gpurun_out/bench_8m.log 2>&1
timeout 600 python bench.py --policy maxpressure --no-cpu > gpurun_out/bench_mp.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 python scripts/bench_batched.py > gpurun_out/bench_batched.log 2>&1
timeout 600 python scripts/floor_and_peaks.py > gpurun_out/floor.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --preroll 10 --no-cpu > gpurun_out/bench_ncu.log 2>&1
tail -n 2 gpurun_out/bench*.log gpurun_out/floor.log
# profiles/ written on the box travel back through gpurun_out/
mkdir -p gpurun_out/profiles && cp profiles/${R}_kstep_ncu_full*.txt profiles/ncu_kstep_traffic*.json gpurun_out/profiles/
