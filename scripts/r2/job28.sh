set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt28.log 2>&1; tail -2 gpurun_out/pt28.log
CC_LIBCC_PATH=build/var/libcc_pb2.so timeout 900 python -m pytest tests/test_gpu_static.py -x -q -k "bit_exact_small or repeat_stress or huge" > gpurun_out/pt28b.log 2>&1; tail -2 gpurun_out/pt28b.log
bash scripts/r2/ab.sh r2ab21 "cur pb2 pb4" "4 3 2"
echo done
