cd ${GRAFT_REPO_ROOT:-/root/repo}
export PREROLL=200
timeout 600 ncu --set full --clock-control none -k regex:k_step -s 210 -c 1 -o gpurun_out/prof_r01 -f bash scripts/time_r01.sh > gpurun_out/ncu_r01.log 2>&1
ncu -i gpurun_out/prof_r01.ncu-rep --page raw --csv > gpurun_out/r01_raw.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/r01_kstep_ncu.txt > /dev/null 2>&1
cat gpurun_out/r01_kstep_ncu.txt
