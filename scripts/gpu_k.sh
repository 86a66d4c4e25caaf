for k in 1 3 4; do for c in 4 3 2; do timeout 300 python bench.py --config $c --k $k --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/k${k}_$c.json 2>> gpurun_out/k.err; done; done
for c in 4 3 2; do timeout 300 python bench.py --config $c --variant hybrid --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/hyb_$c.json 2>> gpurun_out/k.err; done
echo done
