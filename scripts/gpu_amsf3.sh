set -x
timeout 900 python -m pytest tests/test_gpu_amsf.py -x -q > gpurun_out/pytest_amsf.log 2>&1; tail -2 gpurun_out/pytest_amsf.log
timeout 1500 python bench.py --amsf --steps 3 --warmup 1 > gpurun_out/amsf_study.json 2> gpurun_out/amsf_study.err
for v in anc256 anc16; do CC_LIBCC_PATH=$PWD/build/var/libcc_$v.so timeout 900 python scripts/probe/amsf_once.py 4 0 5 > gpurun_out/amsf_$v.log 2>&1; done
timeout 900 python scripts/probe/amsf_once.py 4 0 5 > gpurun_out/amsf_main.log 2>&1
echo done
