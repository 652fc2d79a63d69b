#!/bin/bash
# Build-flag A/B on the GPU box: for each LCX_NVCC_EXTRA variant, a clean build and a short
# bench (per-stage ms).  usage: bash tools/variants.sh "" "-DFOO=1" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  LCX_NVCC_EXTRA="$v" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-extra > /tmp/v.json 2>/tmp/v.err
  python -c "
import json,sys;d=json.loads(open('/tmp/v.json').read().strip().splitlines()[-1])
print('%-40s'%sys.argv[1], round(d['ms_per_step'],1), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" "[$v]" || tail -3 /tmp/v.err
done
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
