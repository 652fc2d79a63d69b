#!/bin/bash
# One GPU-box session: smoke, the 128K config test alone, the full -m gpu suite, a bench
# line.  Logs -> gpurun_out/.  usage: bash tools/gpu_round.sh [tests|bench|all]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what=${1:-all}
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/nproc.txt
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
if [ "$what" != bench ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x -n 4 --timeout 900 -p no:cacheprovider \
      > gpurun_out/gputest.log 2>&1
  echo "gpu tests rc=$?"
  tail -5 gpurun_out/gputest.log
fi
if [ "$what" != tests ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"
  tail -c 1500 gpurun_out/bench.json
fi
