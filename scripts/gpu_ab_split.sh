set -x
for i in 1 2; do
for c in 4 3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sp_main_${c}_$i.json 2>> gpurun_out/sp.err
  CC_LIBCC_PATH=$PWD/build/var/libcc_nosplit.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sp_nosplit_${c}_$i.json 2>> gpurun_out/sp.err
done
done
echo done
