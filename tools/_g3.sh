free -g > gpurun_out/free.txt
bash tools/gpu_round.sh all
timeout 600 ncu --set full --clock-control none --import-source on -k regex:est_tc_kernel -s 40 -c 2 \
   -o gpurun_out/prof_est python tools/run_once.py 1048576 1000 6096 > gpurun_out/ncu_est.log 2>&1
echo ncu rc=$?
