# round-end style set (outputs in gpurun_out/${1:-round}): smoke, pytest -m gpu, the default
# bench line (with the oracle on the full C4 graph), the reference arm, C1 (CUDA graph) - C3 and
# C5 lines, the NEXT-2/NEXT-4 studies, then the ncu launch list and one full capture of the
# default command (each only after that command exited 0 without ncu)
set -x
D=gpurun_out/${1:-round}; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
timeout 1200 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > $D/bench_c5.json 2> $D/bench_c5.err
timeout 600 python bench.py --config 1 --graph --steps 50 > $D/bench_c1_graph.json 2> $D/bench_c1_graph.err
for c in 1 2 3; do timeout 900 python bench.py --config $c > $D/bench_c$c.json 2> $D/bench_c$c.err; done
timeout 1800 python bench.py --amsf --steps 3 --warmup 1 > $D/amsf.json 2> $D/amsf.err
timeout 1800 python bench.py --incr-sweep > $D/incr_sweep.json 2> $D/incr_sweep.err
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > $D/incr_latency.txt 2>&1
P="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $P > $D/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches_c4.csv $P > $D/ncu_l.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending|k_link_refill|k_sample_init|k_finish|k_relabel|k_identify|k_probe|k_compress" --launch-skip 21 -c 10 -o $D/c4_full $P > $D/ncu_f.log 2>&1
echo done
