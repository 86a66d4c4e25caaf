timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -2
for v in main IL8 SEQ; do
  if [ $v = main ]; then unset CC_LIBCC_PATH; else export CC_LIBCC_PATH=$PWD/build/var/libcc_$v.so; fi
  for c in 4 3 2 1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$c.json 2>> gpurun_out/ab.err; done
done
echo done
