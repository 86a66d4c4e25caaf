# ncu launch lists (time + DRAM bytes) of C1-C3, their per-call DRAM bytes merged into
# profiles/ncu_traffic.json, then the C1-C3 bench lines (which read it) re-run
D=gpurun_out/${1:-traffic}; mkdir -p $D
for c in 1 2 3; do
  P="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $P > $D/plain_c$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches_c$c.csv $P > $D/ncu_c$c.log 2>&1
done
python scripts/launches_traffic.py $D/launches_c1.csv C1-er-100k 3 > $D/per_call.txt 2>&1
python scripts/launches_traffic.py $D/launches_c2.csv C2-grid-4096 3 >> $D/per_call.txt 2>&1
python scripts/launches_traffic.py $D/launches_c3.csv C3-rmat-24 3 >> $D/per_call.txt 2>&1
cp profiles/ncu_traffic.json $D/ncu_traffic.json
for c in 1 2 3; do timeout 900 python bench.py --config $c > $D/bench_c$c.json 2> $D/bench_c$c.err; done
timeout 600 python bench.py --config 1 --graph --steps 50 > $D/bench_c1_graph.json 2> $D/bench_c1_graph.err
echo done
