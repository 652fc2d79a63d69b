#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the smoke test and
# the small tcgen05 / estimator / selection parity cases.  Logs -> gpurun_out/sanitize_*.log
# usage (on the GPU box): bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE="python -c 'import __graft_entry__ as g; g.smoke()'"
CASES="python tools/sanitize_cases.py"
for tool in memcheck racecheck synccheck initcheck; do
  for what in smoke cases; do
    cmd=$SMOKE; [ $what = cases ] && cmd=$CASES
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    [ $tool = initcheck ] && extra=""
    echo "== $tool $what" | tee -a gpurun_out/sanitize_summary.txt
    timeout 420 bash -c "$CS --tool $tool $extra --target-processes all --print-limit 50 \
        --error-exitcode 99 $cmd" > gpurun_out/sanitize_${tool}_${what}.log 2>&1
    rc=$?
    echo "rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${what}.log | tail -3 | tr '\n' ' ')" \
      | tee -a gpurun_out/sanitize_summary.txt
  done
done
