# NEXT-4 AMSF parity + the static suite after the cc_common refactor
set -x
timeout 900 python -m pytest tests/test_gpu_gen.py tests/test_gpu_amsf.py -x -q > gpurun_out/pytest_amsf.log 2>&1; tail -5 gpurun_out/pytest_amsf.log
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_full.py -x -q -k amsf -s > gpurun_out/pytest_amsf_full.log 2>&1; tail -5 gpurun_out/pytest_amsf_full.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
echo done
