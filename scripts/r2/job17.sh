set -x
timeout 900 python -m pytest tests/test_gpu_incr.py tests/test_gpu_static.py -x -q > gpurun_out/pt17.log 2>&1; tail -2 gpurun_out/pt17.log
D=gpurun_out/r2ab12; mkdir -p $D
for rep in 1 2 3; do for v in cur prevq; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/c5_${v}_$rep.json 2> $D/c5_${v}_$rep.err
done; done
for v in cur prevq; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 4 --flags 65536 --steps 10 --no-e2e --no-cpu-baseline > $D/c4fused_${v}.json 2> $D/c4fused_${v}.err
done
echo done
