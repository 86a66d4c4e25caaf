# full ncu captures (source-level) of k_link_pending on C3 and C4
D=gpurun_out/j34; mkdir -p $D
for c in 3 4; do
P="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $P > $D/plain_c$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending" --launch-skip 4 -c 1 -o $D/c${c}_link $P > $D/ncu_c$c.log 2>&1
done
echo done
