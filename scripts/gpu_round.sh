# round-end style: smoke, tests, default bench, reference arm, C5, ncu launch list + full capture
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
P="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $P > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_l.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_link_refill|k_sample_init|k_finish|k_compress|k_identify|k_probe" -c 10 -o gpurun_out/prof_full $P > gpurun_out/ncu_f.log 2>&1
echo done
