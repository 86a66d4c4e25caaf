timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -2
for c in 4 3 2 1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_$c.json 2>> gpurun_out/q.err; done
echo done
