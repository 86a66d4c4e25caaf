set -x
D=gpurun_out/r2ab8; mkdir -p $D
for rep in 1 2; do for v in cur lrbranchy; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $D/c5_${v}_$rep.json 2> $D/c5_${v}_$rep.err
  env $L timeout 600 python bench.py --config 4 --k 0 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $D/c4k0_${v}_$rep.json 2> $D/c4k0_${v}_$rep.err
  env $L timeout 600 python bench.py --config 2 --k 0 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $D/c2k0_${v}_$rep.json 2> $D/c2k0_${v}_$rep.err
done; done
echo done
