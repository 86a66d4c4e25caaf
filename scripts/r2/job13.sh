set -x
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/pt13.log 2>&1; tail -2 gpurun_out/pt13.log
bash scripts/r2/ab.sh r2ab9 "cur pe1 big512" "4 3 2"
for v in cur pe1 big512; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 python bench.py --config 4 --k 0 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r2ab9/c4k0_$v.json 2> gpurun_out/r2ab9/c4k0_$v.err
  env $L timeout 600 python bench.py --config 2 --k 0 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r2ab9/c2k0_$v.json 2> gpurun_out/r2ab9/c2k0_$v.err
done
echo done
