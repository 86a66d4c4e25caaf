# ncu --set full of the C5 kernels (one cc_incr_batches call, mid-stream batch) and of one C3 / C2
# labels call on the last code, exported as raw CSV
D=gpurun_out/${1:-ncu53f}; mkdir -p $D
P5="python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 1 --warmup 1"
timeout 300 $P5 > $D/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_insert|k_query" --launch-skip 200 -c 2 -o $D/c5_full $P5 > $D/ncu_c5.log 2>&1
ncu -i $D/c5_full.ncu-rep --page raw --csv > $D/c5_full_raw.csv 2>/dev/null
for c in 3 2; do
  P="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 300 $P > $D/plain_c$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending|k_link_refill|k_sample_init|k_finish|k_relabel|k_compress|k_probe|k_identify" --launch-skip 22 -c 11 -o $D/c${c}_full $P > $D/ncu_c$c.log 2>&1
  ncu -i $D/c${c}_full.ncu-rep --page raw --csv > $D/c${c}_full_raw.csv 2>/dev/null
done
rm -f $D/*.ncu-rep
echo done
