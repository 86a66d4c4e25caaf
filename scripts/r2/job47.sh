# k_insert at 128 threads (default now); k_query block 128 / 64 variants; C5 A/B
mkdir -p gpurun_out/j47
timeout 900 python -m pytest tests/test_gpu_incr.py -x -q > gpurun_out/j47/incr.log 2>&1; echo "rc=$?" >> gpurun_out/j47/incr.log
mkdir -p gpurun_out/j47
for rep in 1 2; do for v in cur qb128 qb64; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j47/c5_${v}_$rep.json 2> gpurun_out/j47/c5_${v}_$rep.err
done; done
echo done
