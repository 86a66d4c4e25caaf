# session re-entry check: smoke, pytest -m gpu, the default bench line
D=gpurun_out/${1:-verify}; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; tail -c 300 $D/bench_default.json
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > $D/bench_c5.json 2> $D/bench_c5.err
echo done
