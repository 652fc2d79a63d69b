#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 90 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -x -n 4 --timeout 600 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputest.log
bash tools/variants_kind.sh planted 3 "" "-DLCX_TC_QK2=0" "" "-DLCX_TC_QK2=0"
bash tools/_r2n.sh
