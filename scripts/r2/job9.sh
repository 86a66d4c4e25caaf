set -x
D=gpurun_out/r2j9; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.log 2>&1; tail -3 $D/pytest_gpu.log
make probes > /dev/null 2>&1; ./scripts/probe/incr_latency 4000 > $D/incr_latency.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B --config 1 --steps 20 --graph > $D/c1_graph.json 2> $D/c1_graph.err
for c in 2 4; do for k in 0 2; do for f in 512 8192 0; do
  timeout 900 $B --config $c --k $k --steps 3 --warmup 3 --flags $f > $D/c${c}_k${k}_f$f.json 2> $D/c${c}_k${k}_f$f.err
done; done; done
P="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $P > $D/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $D/launches_c4.csv $P > $D/ncu_l.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_link_refill|k_sample_init|k_finish|k_relabel|k_identify|k_probe|k_compress" -c 9 -o $D/c4_full $P > $D/ncu_f.log 2>&1
echo done
