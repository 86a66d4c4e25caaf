set -x
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -3
B="python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/b4.json 2> gpurun_out/b4.err
timeout 600 $B --l2-fetch 32 > gpurun_out/b4_f32.json 2> gpurun_out/b4_f32.err
timeout 600 $B --l2-fetch 128 > gpurun_out/b4_f128.json 2> gpurun_out/b4_f128.err
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err
P="python bench.py --config 4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sample_init|k_link_pending|k_finish|k_compress" -c 5 -o gpurun_out/prof_c4b $P > gpurun_out/ncu2.log 2>&1
echo done
