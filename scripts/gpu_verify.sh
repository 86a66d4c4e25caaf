# quick verification: all GPU tests except the full-size ones, default bench (short), C3/C2
set -x
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in 3 2; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/v_$c.json 2>> gpurun_out/v.err; done
echo done
