set -x
D=gpurun_out/r2ab15; mkdir -p $D
for rep in 1 2; do for c in 4 3 1; do for v in cur lb1 lb2 lb3; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config $c --flags 2048 --steps 10 --no-e2e --no-cpu-baseline > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
done; done; done
echo done
