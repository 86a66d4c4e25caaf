for v in main V1 V2; do
  if [ $v = main ]; then unset CC_LIBCC_PATH; else export CC_LIBCC_PATH=$PWD/build/var/libcc_$v.so; fi
  for c in 4 3 2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${v}_$c.json 2>> gpurun_out/ab.err; done
done
echo done
