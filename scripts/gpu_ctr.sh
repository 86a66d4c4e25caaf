for c in 4 2 3; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ctr_$c.json 2>> gpurun_out/ctr.err; done
echo done
