# A/B: round-1 library vs resident-grid link (this tree) vs MINB=8 variant, C1-C4
set -x
mkdir -p gpurun_out/r2ab1
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 3 4 2 1; do
  for v in r1 cur minb8; do
    if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
    env $L timeout 600 $B --config $c > gpurun_out/r2ab1/c${c}_$v.json 2> gpurun_out/r2ab1/c${c}_$v.err
  done
done
echo done
