set -x
bash scripts/r2/ab.sh r2ab13 "cur si2 kv4m4" "4 3"
D=gpurun_out/r2ab13
for c in 3 2 1; do for f in 0 2048; do
  timeout 600 python bench.py --config $c --flags $f --steps 10 --no-e2e --no-cpu-baseline > $D/c${c}_f$f.json 2> $D/c${c}_f$f.err
done; done
echo done
