timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -3
for c in 4 3 2; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --flags 512 > gpurun_out/sv_$c.json 2>> gpurun_out/sv.err; done
for c in 4 3 2; do timeout 300 python bench.py --config $c --k 0 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --flags 512 > gpurun_out/sv0_$c.json 2>> gpurun_out/sv.err; done
echo done
