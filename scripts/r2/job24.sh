set -x
timeout 900 python -m pytest tests/test_gpu_amsf.py -x -q > gpurun_out/pt24.log 2>&1; tail -2 gpurun_out/pt24.log
D=gpurun_out/r2ab18; mkdir -p $D
for v in cur amsfprev; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 900 python scripts/probe/amsf_once.py 3 0 6 > $D/amsf3_$v.txt 2>&1
  env $L timeout 900 python scripts/probe/amsf_once.py 4 0 6 > $D/amsf4_$v.txt 2>&1
done
echo done
