set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q -k "lmax_forcing" > gpurun_out/pt20.log 2>&1; tail -2 gpurun_out/pt20.log
D=gpurun_out/r2ab14; mkdir -p $D
for c in 4 3 2; do for v in cur lb8 lb2; do for f in 0 2048; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  if [ $v != cur ] && [ $f = 0 ]; then continue; fi
  env $L timeout 600 python bench.py --config $c --flags $f --steps 10 --no-e2e --no-cpu-baseline > $D/c${c}_${v}_f$f.json 2> $D/c${c}_${v}_f$f.err
done; done; done
echo done
