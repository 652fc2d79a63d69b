#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 90 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc; tail -1 gpurun_out/smoke.log
[ $rc -ne 0 ] && exit 1
bash tools/_r2o.sh
