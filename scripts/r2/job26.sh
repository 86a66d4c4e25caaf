set -x
D=gpurun_out/r2j26; mkdir -p $D
bash scripts/r2/ab.sh r2ab19 "cur pf pfns" "4 3"
P4="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
P3="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending" --launch-skip 2 -c 1 -o $D/c4_link $P4 > $D/ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending" --launch-skip 2 -c 1 -o $D/c3_link $P3 > $D/ncu3.log 2>&1
echo done
