# pending links split by v's id range (CC_PEND_SPLIT) on C4: A/B, then full-size C4 parity on the variant
mkdir -p gpurun_out/j53
bash scripts/r2/ab.sh j53 "cur sp" "4"
CC_LIBCC_PATH=build/var/libcc_sp.so timeout 1200 python -m pytest tests/test_gpu_full.py -x -q -k "C4 or no_sampling" > gpurun_out/j53/full_sp.log 2>&1; echo "rc=$?" >> gpurun_out/j53/full_sp.log
