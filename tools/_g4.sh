set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "line_scores or estimate or select or sharded or smoke" -p no:cacheprovider > gpurun_out/t4.log 2>&1; echo t4 rc=$?; tail -2 gpurun_out/t4.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra > gpurun_out/bench4.json 2>gpurun_out/bench4.err; echo bench rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench4.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['clocks']); print({k:v['ms_per_step'] for k,v in d['kernels'].items()})"
LCX_NVCC_EXTRA=-DLCX_TC_WAITPROF python -m paper_2501_15383_b200.build --clean > /dev/null 2>&1
timeout 300 python tools/trace_wait.py > gpurun_out/waitprof.txt 2>&1; echo wp rc=$?; cat gpurun_out/waitprof.txt
