# SV / CRFA: tested-writeMin + shared-memory append buffers; static tests, then C4/C2 k=0 and k=2 vs the previous build
mkdir -p gpurun_out/j42
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j42/static.log 2>&1; echo "rc=$?" >> gpurun_out/j42/static.log
for c in 4 2; do for k in 0 2; do for f in 512 8192; do for v in cur old; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 900 python bench.py --config $c --k $k --flags $f --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j42/c${c}_k${k}_f${f}_$v.json 2> gpurun_out/j42/c${c}_k${k}_f${f}_$v.err
done; done; done; done
echo done
