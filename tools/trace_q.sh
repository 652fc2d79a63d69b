#!/bin/bash
# Per-quadrant softmax timeline (tools/trace_q.py) of a trace build.  usage: bash tools/trace_q.sh [extra flags]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LCX_NVCC_EXTRA="-DLCX_TC_TRACE -DLCX_TC_TRACE_SM -DLCX_TC_TRACE_Q $*" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1 || echo build failed
timeout 120 python tools/trace_q.py > gpurun_out/trace_q.txt 2>&1; echo rc=$?
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
