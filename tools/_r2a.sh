#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for tool in synccheck racecheck; do
  timeout 600 $CS --tool $tool --print-limit 20 --error-exitcode 99 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/san_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_smoke.log | tail -1)"
done
timeout 900 $CS --tool synccheck --print-limit 20 --error-exitcode 99 python tools/sanitize_cases.py > gpurun_out/san_synccheck_cases.log 2>&1
echo "synccheck cases rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/san_synccheck_cases.log | tail -1)"
bash tools/_wp.sh
timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --kind planted > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; echo bench rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_x.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items()}, d['clocks'])
print(json.dumps(d['scattered_inputs'], indent=1))"
