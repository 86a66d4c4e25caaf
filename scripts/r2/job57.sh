# k_sv_copy entries per lane per sweep (CC_SV_R 1 / 2 / 4=cur): C4 k=0 SV / CRFA, static tests on cur
mkdir -p gpurun_out/j57
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j57/static.log 2>&1; echo "rc=$?" >> gpurun_out/j57/static.log
for f in 512 8192; do for v in cur svr1 svr2; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 900 python bench.py --config 4 --k 0 --flags $f --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j57/c4_k0_f${f}_$v.json 2> gpurun_out/j57/c4_k0_f${f}_$v.err
done; done
