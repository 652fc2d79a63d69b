#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
bash tools/variants.sh "-DLCX_TC_MERGE=0" "" "-DLCX_TC_MERGE=0" ""
for tool in synccheck racecheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/san_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_smoke.log | tail -1)"
done
bash tools/_wp.sh
