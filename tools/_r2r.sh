#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LCX_NVCC_EXTRA="$1" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
timeout 90 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc; tail -1 gpurun_out/smoke.log
[ $rc -ne 0 ] && exit 1
bash tools/variants_kind.sh planted 3 "$1" "" "$1"
LCX_NVCC_EXTRA="-DLCX_TC_TRACE -DLCX_TC_TRACE_SM -DLCX_TC_TRACE_Q $1" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
timeout 120 python tools/trace_q.py > gpurun_out/trace_q.txt 2>&1; echo trace rc=$?
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
