set -x
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -5
for c in 4 3 2; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b$c.json 2> gpurun_out/b$c.err
done
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags 64 > gpurun_out/b4_nomid.json 2> gpurun_out/b4_nomid.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --k 0 > gpurun_out/b4_k0.json 2> gpurun_out/b4_k0.err
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --flags 64 > gpurun_out/b2_nomid.json 2> gpurun_out/b2_nomid.err
timeout 900 python -m pytest tests/test_gpu_full.py -x -q 2>&1 | tail -3
echo done
