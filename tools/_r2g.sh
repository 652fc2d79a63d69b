#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1m.csv python tools/run_once.py 1048576 1000 6096 > gpurun_out/ncu_l.log 2>&1; echo l rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:est_tc_kernel -s 58 -c 2 \
   -o gpurun_out/prof_est python tools/run_once.py 1048576 1000 6096 > gpurun_out/ncu_est.log 2>&1; echo e rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_gather_kernel -s 29 -c 1 \
   -o gpurun_out/prof_gather python tools/run_once.py 1048576 1000 6096 iid > gpurun_out/ncu_g.log 2>&1; echo g rc=$?
