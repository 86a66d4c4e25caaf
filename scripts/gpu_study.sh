timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -2
timeout 1200 python bench.py --study --steps 5 --warmup 2 > gpurun_out/study.json 2> gpurun_out/study.err
echo done
