# round-0 hook under the smaller of the first two samples (CC_HOOK2): static tests on the variant, A/B
mkdir -p gpurun_out/j40
CC_LIBCC_PATH=build/var/libcc_h2.so timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j40/static_h2.log 2>&1; echo "rc=$?" >> gpurun_out/j40/static_h2.log
bash scripts/r2/ab.sh j40 "cur h2" "3 4 1 2"
