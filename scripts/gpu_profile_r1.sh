set -x
timeout 600 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_full.py 2>&1 | tail -5
B="python bench.py --config 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
timeout 300 python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b3.json 2> gpurun_out/b3.err
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $B > gpurun_out/ncu1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sample_init|k_link_pending|k_compress|k_finish" -c 7 -o gpurun_out/prof_c4 $B > gpurun_out/ncu2.log 2>&1
echo done
