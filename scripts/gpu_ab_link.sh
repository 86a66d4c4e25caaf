# A/B of the k-out link variants: contracted (default), in-place refill, in-place round-1 kernel
set -x
timeout 600 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pytest_static.log 2>&1; tail -2 gpurun_out/pytest_static.log
for c in 4 3 2; do
  for f in 0 1024 3072; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags $f > gpurun_out/ab_f${f}_$c.json 2>> gpurun_out/ab.err
  done
  CC_LIBCC_PATH=$PWD/build/var/libcc_rf8.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags 1024 > gpurun_out/ab_rf8_$c.json 2>> gpurun_out/ab.err
done
echo done
