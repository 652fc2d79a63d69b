#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/variants.sh "-DLCX_TC_HEAD_MAJOR" "" "-DLCX_TC_HEAD_MAJOR" ""
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 58 -c 2 \
   -o gpurun_out/prof_attn python tools/run_once.py 1048576 1000 6096 > gpurun_out/ncu_attn.log 2>&1
echo ncu rc=$?
timeout 1500 python -m pytest tests -m gpu -q -x -n 4 --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/gputest.log
