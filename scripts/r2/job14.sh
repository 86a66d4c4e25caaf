set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt14.log 2>&1; tail -2 gpurun_out/pt14.log
D=gpurun_out/r2ab10; mkdir -p $D
for rep in 1 2; do for v in cur pe1; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 2 --k 0 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $D/c2k0_${v}_$rep.json 2> $D/c2k0_${v}_$rep.err
  env $L timeout 600 python bench.py --config 4 --steps 10 --no-e2e --no-cpu-baseline > $D/c4_${v}_$rep.json 2> $D/c4_${v}_$rep.err
  env $L timeout 600 python bench.py --config 3 --steps 10 --no-e2e --no-cpu-baseline > $D/c3_${v}_$rep.json 2> $D/c3_${v}_$rep.err
done; done
echo done
