#!/bin/bash
# Build-flag A/B on the GPU box for one input kind: per variant a clean build and a short
# bench (per-stage ms).  usage: bash tools/variants_kind.sh KIND STEPS "" "-DFOO=1" ...
cd "$(dirname "$0")/.."
kind=$1; steps=$2; shift 2
for v in "$@"; do
  LCX_NVCC_EXTRA="$v" python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 240 python bench.py --kind $kind --steps $steps --warmup 1 --no-e2e --no-cpu --no-extra > /tmp/v.json 2>/tmp/v.err
  python -c "
import json,sys;d=json.loads(open('/tmp/v.json').read().strip().splitlines()[-1])
print('%-8s %-36s'%(sys.argv[2], sys.argv[1]), round(d['ms_per_step'],1), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" "[$v]" $kind || tail -3 /tmp/v.err
done
python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
