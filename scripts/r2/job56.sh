# SV / CRFA edge copy with long lists split into pieces (k_sv_pieces): static tests, C4 k=0 SV/CRFA timings
mkdir -p gpurun_out/j56
timeout 900 python -m pytest tests/test_gpu_static.py -x -q > gpurun_out/j56/static.log 2>&1; echo "rc=$?" >> gpurun_out/j56/static.log
for f in 512 8192; do
  timeout 900 python bench.py --config 4 --k 0 --flags $f --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j56/c4_k0_f$f.json 2> gpurun_out/j56/c4_k0_f$f.err
done
timeout 1400 python -m pytest tests/test_gpu_full.py -x -q -k "no_sampling" > gpurun_out/j56/full.log 2>&1; echo "rc=$?" >> gpurun_out/j56/full.log
