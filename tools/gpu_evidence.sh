#!/bin/bash
# Round evidence on one GPU box: sanitizers, C4 recall sweep (256K, planted + structured),
# C5 stack (1M, 28 layers, planted; iid with fewer layers) next to dense SDPA and the
# repo's own dense DCA path.  Logs -> gpurun_out/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what=${1:-all}
if [ "$what" = all ] || [ "$what" = sanitize ]; then
  bash tools/sanitize.sh > gpurun_out/sanitize.out 2>&1; echo "sanitize rc=$?"
  cat gpurun_out/sanitize_summary.txt
fi
if [ "$what" = all ] || [ "$what" = c4 ]; then
  timeout 1200 python tools/recall_sweep.py 262144 planted > gpurun_out/recall_sweep_planted.jsonl 2> gpurun_out/recall_sweep.err
  echo "c4 rc=$?"; tail -2 gpurun_out/recall_sweep_planted.jsonl
fi
if [ "$what" = all ] || [ "$what" = c5 ]; then
  timeout 1500 python tools/stack_bench.py 1048576 28 planted > gpurun_out/stack_planted.json 2> gpurun_out/stack_planted.err
  echo "c5 planted rc=$?"; tail -c 600 gpurun_out/stack_planted.json; tail -3 gpurun_out/stack_planted.err
  timeout 1500 python tools/stack_bench.py 1048576 4 iid > gpurun_out/stack_iid.json 2> gpurun_out/stack_iid.err
  echo "c5 iid rc=$?"; tail -c 600 gpurun_out/stack_iid.json; tail -3 gpurun_out/stack_iid.err
fi
