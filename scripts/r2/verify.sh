# quick round-2 verification: static GPU tests + C1-C4 bench lines (no e2e / cpu leg)
set -x
D=gpurun_out/${1:-r2v}
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > $D/pytest_static.log 2>&1; tail -3 $D/pytest_static.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 4 3 2 1; do timeout 600 $B --config $c > $D/c$c.json 2> $D/c$c.err; done
echo done
