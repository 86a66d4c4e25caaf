# final check of the last code: smoke + the whole GPU suite + the default bench line
D=gpurun_out/${1:-vfinal}; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -n 2 $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -n 3 $D/pytest_gpu.log
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err
python -c "import json;d=json.load(open('$D/bench_default.json'));print(d['value'],d['ms_per_step'],d['finish']['t_fin_ms'],d['parity'])"
echo done
