set -x
timeout 900 python -m pytest tests/test_gpu_incr.py tests/test_gpu_static.py -x -q > gpurun_out/pt6.log 2>&1; tail -2 gpurun_out/pt6.log
bash scripts/r2/ab.sh r2ab4 "cur persist persist5 persist8" "4 3"
mkdir -p gpurun_out/r2c5
for v in cur r1; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2c5/c5_$v.json 2> gpurun_out/r2c5/c5_$v.err
done
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > gpurun_out/r2c5/incr_latency.txt 2>&1
echo done
