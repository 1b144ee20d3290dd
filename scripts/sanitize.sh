#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over a short
# run of every library kernel (scripts/sanitize_run.py); summaries in gpurun_out/
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py \
      > gpurun_out/sanitizer_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -n 4 gpurun_out/sanitizer_$tool.log
done
