# per-lane streaming link (k_link_stream) vs k_link_pending: static tests on the variant, A/B C3/C4/C1
mkdir -p gpurun_out/j36
CC_LIBCC_PATH=build/var/libcc_st8.so timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j36/static_st8.log 2>&1; echo "rc=$?" >> gpurun_out/j36/static_st8.log
bash scripts/r2/ab.sh j36 "cur st8 st6" "3 4 1"
