# A/B of build variants: bash scripts/r2/ab.sh OUTDIR "cur fin6 ..." "4 3" [extra bench args]
# cur = the in-tree libcc.so; NAME = build/var/libcc_NAME.so.  Variants alternate per config.
set -x
D=gpurun_out/$1; mkdir -p $D
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 $4"
for c in $3; do
  for rep in 1 2; do
    for v in $2; do
      if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
      env $L timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
    done
  done
done
echo done
