set -x
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -3
B="python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/b4.json 2> gpurun_out/b4.err
for c in 3 2 1; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err; done
timeout 600 python bench.py --config 5 --steps 3 --warmup 1 > gpurun_out/b5.json 2> gpurun_out/b5.err
echo done
