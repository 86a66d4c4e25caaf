set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt32.log 2>&1; tail -2 gpurun_out/pt32.log
bash scripts/r2/ab.sh r2ab23 "cur rlprev" "4 3 2"
echo done
