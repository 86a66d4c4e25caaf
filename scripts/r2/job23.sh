set -x
D=gpurun_out/r2ab17; mkdir -p $D
for rep in 1 2; do for f in 0 2048 64 2112; do
  timeout 600 python bench.py --config 2 --flags $f --steps 10 --no-e2e --no-cpu-baseline > $D/c2_f${f}_$rep.json 2> $D/c2_f${f}_$rep.err
done; done
for f in 0 2048; do timeout 600 python bench.py --config 5 --flags $f --steps 3 --no-e2e --no-cpu-baseline > $D/c5_f$f.json 2> $D/c5_f$f.err; done
echo done
