# contracted k-out link: parity + A/B against the in-place link
set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pytest_static.log 2>&1; tail -3 gpurun_out/pytest_static.log
for c in 4 3 2 1; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ct_$c.json 2>> gpurun_out/ct.err
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags 1024 > gpurun_out/nc_$c.json 2>> gpurun_out/ct.err
done
echo done
