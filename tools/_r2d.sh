#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python tools/run_once.py 131072 1000 6096 > gpurun_out/ncu_small.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_small.log; cut -d, -f5 gpurun_out/launches_small.csv | sort | uniq -c | sort -rn | head -30
