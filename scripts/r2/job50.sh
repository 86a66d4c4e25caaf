# C1: does a mid compress before k_link_pending pay when the pending links fit in one wave?
D=gpurun_out/j50; mkdir -p $D
for rep in 1 2; do for f in 0 128 2176 2048; do
  timeout 300 python bench.py --config 1 --flags $f --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $D/c1_f${f}_$rep.json 2> $D/c1_f${f}_$rep.err
done; done
echo done
