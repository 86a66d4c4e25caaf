set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt22.log 2>&1; tail -2 gpurun_out/pt22.log
D=gpurun_out/r2ab16; mkdir -p $D
for rep in 1 2; do for c in 4 3 2 1; do for f in 0 262144; do
  timeout 600 python bench.py --config $c --flags $f --steps 10 --no-e2e --no-cpu-baseline > $D/c${c}_f${f}_$rep.json 2> $D/c${c}_f${f}_$rep.err
done; done; done
echo done
