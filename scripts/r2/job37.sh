# lane-refill link with one predicated memory op per iteration (CC_REFILL_ONEOP) vs the current refill and k_link_pending
mkdir -p gpurun_out/j37
CC_LIBCC_PATH=build/var/libcc_r1m6.so timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j37/static_r1m6.log 2>&1; echo "rc=$?" >> gpurun_out/j37/static_r1m6.log
bash scripts/r2/ab.sh j37/refill "cur r1m6 r0m8 r1m8" "3 4" "--flags 262144"
bash scripts/r2/ab.sh j37/dflt "cur r1m6" "2"
