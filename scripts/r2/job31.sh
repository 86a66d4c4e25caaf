set -x
timeout 900 python -m pytest tests/test_gpu_static.py tests/test_gpu_amsf.py -x -q > gpurun_out/pt31.log 2>&1; tail -2 gpurun_out/pt31.log
D=gpurun_out/r2sf; mkdir -p $D
for v in cur sfprev; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python scripts/r2/sf_ab.py 4 10 > $D/c4_$v.txt 2>&1
  env $L timeout 600 python scripts/r2/sf_ab.py 3 10 > $D/c3_$v.txt 2>&1
done
echo done
