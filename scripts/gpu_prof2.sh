P="python bench.py --config 4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending|k_sample_init|k_finish$|k_finish<|k_compress" -c 5 -o gpurun_out/prof_c4c $P > gpurun_out/ncu3.log 2>&1
echo done
