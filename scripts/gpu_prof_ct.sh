# ncu of the contracted vs in-place link kernels (C3 and C4)
set -x
B3="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
B4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $B3 > gpurun_out/p3.log 2>&1 && timeout 300 $B4 > gpurun_out/p4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link|k_compress|k_rank|k_contract|k_finish<" -c 7 -o gpurun_out/prof_ct3 $B3 > gpurun_out/ncu_ct3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link|k_compress|k_rank|k_contract|k_finish<" -c 7 -o gpurun_out/prof_ct4 $B4 > gpurun_out/ncu_ct4.log 2>&1
echo done
