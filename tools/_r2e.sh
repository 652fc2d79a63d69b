#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 29 -c 1 \
   -o gpurun_out/prof_attn python tools/run_once.py 1048576 1000 6096 > gpurun_out/ncu_attn.log 2>&1
echo ncu rc=$?; tail -2 gpurun_out/ncu_attn.log; ls -la gpurun_out/prof_attn*
