# AMSF carry-list appends through WarpBuf: amsf tests, then the --amsf study vs the previous build
mkdir -p gpurun_out/j43
timeout 1200 python -m pytest tests/test_gpu_amsf.py -x -q > gpurun_out/j43/amsf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/j43/amsf_tests.log
timeout 1200 python bench.py --amsf --steps 3 --warmup 1 > gpurun_out/j43/amsf_cur.json 2> gpurun_out/j43/amsf_cur.err
CC_LIBCC_PATH=build/var/libcc_prevamsf.so timeout 1200 python bench.py --amsf --steps 3 --warmup 1 > gpurun_out/j43/amsf_prev.json 2> gpurun_out/j43/amsf_prev.err
echo done
