#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/_wp.sh
bash tools/variants.sh "" "-DLCX_TC_LANE_ARRIVE=1" ""
LCX_NVCC_EXTRA="-DLCX_TC_LANE_ARRIVE=1" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 99 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/san_racecheck_smoke.log 2>&1
echo "racecheck(lane arrive) smoke rc=$? $(grep -E 'RACECHECK SUMMARY' gpurun_out/san_racecheck_smoke.log | tail -1)"
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
