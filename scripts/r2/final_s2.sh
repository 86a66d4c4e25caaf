# final round-2 set after the k_finish_proc split (outputs in gpurun_out/$1): smoke, pytest -m gpu,
# ncu launch lists of C1-C4 -> profiles/ncu_traffic.json (on the box, copied out), the bench lines
# (which read it), one ncu --set full capture of the C4 call + counter table, then the studies
set -x
D=gpurun_out/${1:-final}; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -n 2 $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -n 3 $D/pytest_gpu.log
for c in 1 2 3 4; do
  P="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $P > $D/plain_c$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches_c$c.csv $P > $D/ncu_l_c$c.log 2>&1
done
python scripts/launches_traffic.py $D/launches_c1.csv C1-er-100k 3 > $D/per_call.txt 2>&1
python scripts/launches_traffic.py $D/launches_c2.csv C2-grid-4096 3 >> $D/per_call.txt 2>&1
python scripts/launches_traffic.py $D/launches_c3.csv C3-rmat-24 3 >> $D/per_call.txt 2>&1
python scripts/launches_traffic.py $D/launches_c4.csv C4-rmat-27 3 >> $D/per_call.txt 2>&1
cp profiles/ncu_traffic.json $D/ncu_traffic.json
timeout 1200 python bench.py > $D/bench_default.json 2> $D/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > $D/bench_c5.json 2> $D/bench_c5.err
timeout 600 python bench.py --config 1 --graph --steps 50 > $D/bench_c1_graph.json 2> $D/bench_c1_graph.err
for c in 1 2 3; do timeout 900 python bench.py --config $c > $D/bench_c$c.json 2> $D/bench_c$c.err; done
P="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending|k_link_refill|k_sample_init|k_finish|k_relabel|k_identify|k_probe|k_compress" --launch-skip 22 -c 11 -o $D/c4_full $P > $D/ncu_f.log 2>&1
ncu -i $D/c4_full.ncu-rep --page raw --csv > $D/c4_full_raw.csv 2>/dev/null
python scripts/ncu_counters.py $D/c4_full_raw.csv > $D/counters_c4.txt 2>&1
timeout 1800 python bench.py --amsf --steps 3 --warmup 1 > $D/amsf.json 2> $D/amsf.err
timeout 1800 python bench.py --incr-sweep > $D/incr_sweep.json 2> $D/incr_sweep.err
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > $D/incr_latency.txt 2>&1
echo done
