# incremental insert on one resident grid-strided wave (CC_INSERT_RESIDENT): incr tests on the variant, C5 A/B
mkdir -p gpurun_out/j46
for rep in 1 2; do for v in cur ib128 ib64; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j46/c5_${v}_$rep.json 2> gpurun_out/j46/c5_${v}_$rep.err
done; done
echo done
