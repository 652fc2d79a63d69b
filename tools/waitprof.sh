#!/bin/bash
# attn_tc wait profile (per role / per softmax phase) on the GPU box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LCX_NVCC_EXTRA="-DLCX_TC_WAITPROF $*" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1 || echo build failed
timeout 300 python tools/trace_wait.py > gpurun_out/waitprof.txt 2>&1; echo wp rc=$?; cat gpurun_out/waitprof.txt
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
