set -x
timeout 900 python -m pytest tests/test_gpu_static.py tests/test_gpu_incr.py -x -q > gpurun_out/pt15.log 2>&1; tail -2 gpurun_out/pt15.log
D=gpurun_out/r2ab11; mkdir -p $D
for v in cur pe1 pe1big512 pe1big1024; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 2 --k 0 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $D/c2k0_${v}.json 2> $D/c2k0_${v}.err
  env $L timeout 600 python bench.py --config 4 --k 0 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $D/c4k0_${v}.json 2> $D/c4k0_${v}.err
  for rep in 1 2; do
  env $L timeout 600 python bench.py --config 4 --steps 10 --no-e2e --no-cpu-baseline > $D/c4_${v}_$rep.json 2> $D/c4_${v}_$rep.err
  env $L timeout 600 python bench.py --config 3 --steps 10 --no-e2e --no-cpu-baseline > $D/c3_${v}_$rep.json 2> $D/c3_${v}_$rep.err
  done
  env $L timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/c5_${v}.json 2> $D/c5_${v}.err
done
echo done
