# NEXT-3 table (SV / CRFA vs UF-Rem-CAS) on C2 / C4 at k = 0 and 2
D=gpurun_out/j44; mkdir -p $D
for c in 2 4; do for k in 0 2; do for f in 0 512 8192; do
  timeout 900 python bench.py --config $c --k $k --flags $f --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/c${c}_k${k}_f$f.json 2> $D/c${c}_k${k}_f$f.err
done; done; done
python scripts/r2/next3_table.py $D > $D/next3.json
echo done
