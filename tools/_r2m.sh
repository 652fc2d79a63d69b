#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
bash tools/variants_kind.sh planted 3 "" "-DLCX_TC_QBUFS=1" "-DLCX_TC_MERGE=0" ""
bash tools/_r2l.sh
