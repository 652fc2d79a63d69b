#!/bin/bash
# Round evidence for the current build: smoke, GPU tests, bench (7B default + 14B heads),
# reference arm, ncu launch list + full captures of the top kernels, sanitizers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# build from the sources in this snapshot (an in-tree .so built before a later edit would
# otherwise be what runs)
python -m paper_2501_15383_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 90 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc
[ $rc -ne 0 ] && exit 1
timeout 600 python -m pytest tests -m gpu -q -x -n 4 --timeout 300 -p no:cacheprovider > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?"; tail -1 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
timeout 600 python bench.py --hq 40 --hkv 8 --no-extra --no-cpu > gpurun_out/bench_14b_final.json 2> gpurun_out/bench_14b.err; echo bench14 rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra > /dev/null 2>&1; echo launches rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 29 -c 1 -o gpurun_out/prof_attn_final python tools/run_once.py 1048576 1000 6096 > /dev/null 2>&1; echo ncu attn rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:est_tc_kernel -s 58 -c 2 -o gpurun_out/prof_est_final python tools/run_once.py 1048576 1000 6096 > /dev/null 2>&1; echo ncu est rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_gather_diag -s 29 -c 1 -o gpurun_out/prof_gather_final python tools/run_once.py 1048576 1000 6096 > /dev/null 2>&1; echo ncu gather rc=$?
for tool in memcheck racecheck synccheck; do
  timeout 400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/san_${tool}_final.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_final.log | tail -1)"
done
