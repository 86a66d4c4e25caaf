set -x
timeout 900 python -m pytest tests/test_gpu_amsf.py -x -q > gpurun_out/pytest_amsf.log 2>&1; tail -3 gpurun_out/pytest_amsf.log
timeout 900 python -m pytest tests/test_gpu_full.py -x -q -k amsf -s > gpurun_out/pytest_amsf_full.log 2>&1; tail -3 gpurun_out/pytest_amsf_full.log
timeout 1500 python bench.py --amsf --steps 3 --warmup 1 > gpurun_out/amsf_study.json 2> gpurun_out/amsf_study.err
echo done
