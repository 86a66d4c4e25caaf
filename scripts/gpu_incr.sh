timeout 900 python -m pytest tests/test_gpu_incr.py -x -q 2>&1 | tail -2
timeout 1200 python bench.py --incr-sweep > gpurun_out/incr_sweep.json 2> gpurun_out/incr_sweep.err
echo done
