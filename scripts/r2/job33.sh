# k_probe mid-compress rule: static tests, then A/B old vs cur on C1/C3/C4
mkdir -p gpurun_out/j33
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j33/static.log 2>&1; echo "static rc=$?" >> gpurun_out/j33/static.log
bash scripts/r2/ab.sh j33 "old cur" "1 3 4"
