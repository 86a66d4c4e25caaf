# bucketed pending links: parity + A/B
set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pytest_static.log 2>&1; tail -3 gpurun_out/pytest_static.log
for c in 4 3 2 1; do
  for f in 0 8192; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags $f > gpurun_out/bk_f${f}_$c.json 2>> gpurun_out/bk.err
  done
done
echo done
