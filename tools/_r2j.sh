#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -n 4 --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputest.log
bash tools/variants_kind.sh iid 1 ""
bash tools/variants_kind.sh planted 3 ""
