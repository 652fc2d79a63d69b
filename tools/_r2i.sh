#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_gather_diag -s 450 -c 1 \
   -o gpurun_out/prof_gdiag python tools/run_once.py 1048576 1000 6096 iid > gpurun_out/ncu_g.log 2>&1; echo g rc=$?
