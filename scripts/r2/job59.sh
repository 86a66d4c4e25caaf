# two interleaved Rem walks per thread (k_link_pending2, CC_LINK_ILV2): static tests on the variant, A/B
mkdir -p gpurun_out/j59
CC_LIBCC_PATH=build/var/libcc_il2.so timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j59/static_il2.log 2>&1; echo "rc=$?" >> gpurun_out/j59/static_il2.log
bash scripts/r2/ab.sh j59 "cur il2" "3 4 1"
