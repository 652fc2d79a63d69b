timeout 400 python -m pytest tests/test_configs.py -m gpu -q -x -k "config1 or config0" --timeout 380 -p no:cacheprovider > gpurun_out/cfg1.log 2>&1; echo cfg1 rc=$?; tail -3 gpurun_out/cfg1.log
bash tools/gpu_round.sh all
