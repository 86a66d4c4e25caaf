set -x
timeout 900 python -m pytest tests/test_gpu_incr.py -x -q > gpurun_out/pt7.log 2>&1; tail -2 gpurun_out/pt7.log
mkdir -p gpurun_out/r2c5b
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > gpurun_out/r2c5b/incr_latency.txt 2>&1
for rep in 1 2; do for v in cur ib1 ib4 r1; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2c5b/c5_${v}_$rep.json 2> gpurun_out/r2c5b/c5_${v}_$rep.err
done; done
bash scripts/r2/ab.sh r2ab5 "cur ldca" "3 4 2 1"
echo done
