set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt11.log 2>&1; tail -2 gpurun_out/pt11.log
bash scripts/r2/ab.sh r2ab7 "cur branchy" "4 3 2 1"
echo done
