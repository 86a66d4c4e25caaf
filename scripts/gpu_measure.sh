# per-config bench lines + AMSF study + AMSF tests
set -x
timeout 900 python -m pytest tests/test_gpu_amsf.py -x -q > gpurun_out/pytest_amsf.log 2>&1; tail -2 gpurun_out/pytest_amsf.log
for c in 1 2 3; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/m_$c.json 2>> gpurun_out/m.err; done
timeout 1500 python bench.py --amsf --steps 3 --warmup 1 > gpurun_out/amsf_study.json 2> gpurun_out/amsf_study.err
echo done
