#!/bin/bash
# A/B of one build-flag variant against the default on the GPU box: clean build, smoke, the
# -m gpu suite, then interleaved short benches.  usage: bash tools/ab_test.sh "-DFLAG=1"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LCX_NVCC_EXTRA="$1" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
timeout 90 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc; tail -1 gpurun_out/smoke.log
[ $rc -ne 0 ] && exit 1
timeout 600 python -m pytest tests -m gpu -q -x -n 4 --timeout 300 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -2 gpurun_out/gputest.log
bash tools/variants_kind.sh planted 3 "$1" "" "$1" ""
