# ncu --set full of the C5 insert/query kernels (mid-stream batch) and of one C3 / C2 labels call,
# exported as raw CSV for scripts/ncu_counters.py (each command exits 0 without ncu first)
D=gpurun_out/${1:-ncu53}; mkdir -p $D
P5="python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 1 --warmup 1"
timeout 300 $P5 > $D/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_query" --launch-skip 200 -c 2 -o $D/c5_full $P5 > $D/ncu_c5.log 2>&1
ncu -i $D/c5_full.ncu-rep --page raw --csv > $D/c5_full_raw.csv 2>/dev/null
for c in 3 2; do
  P="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $P > $D/plain_c$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending|k_link_refill|k_sample_init|k_finish|k_relabel|k_compress" --launch-skip 18 -c 9 -o $D/c${c}_full $P > $D/ncu_c$c.log 2>&1
  ncu -i $D/c${c}_full.ncu-rep --page raw --csv > $D/c${c}_full_raw.csv 2>/dev/null
done
python scripts/ncu_counters.py $D/c5_full_raw.csv $D/c3_full_raw.csv $D/c2_full_raw.csv > $D/counters.txt 2>&1
rm -f $D/*.ncu-rep.tmp
echo done
