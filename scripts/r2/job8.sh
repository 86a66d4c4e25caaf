set -x
D=gpurun_out/r2j8; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 4 3 2 1; do timeout 600 $B --config $c > $D/c$c.json 2> $D/c$c.err; done
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/c5.json 2> $D/c5.err
for f in 512 8192; do timeout 600 $B --config 4 --k 0 --steps 3 --flags $f > $D/c4_k0_f$f.json 2> $D/c4_k0_f$f.err; done
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > $D/incr_latency.txt 2>&1
echo done
