set -x
bash scripts/r2/ab.sh r2ab6 "cur rgrid0 rminb8 rgrid12 relaxed" "3 4 2 1"
D=gpurun_out/r2ab6
P="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_refill" --launch-skip 2 -c 1 -o $D/c3_link $P > $D/ncu_c3.log 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
timeout 600 $B --config 1 --flags 128 > $D/c1_mid.json 2> $D/c1_mid.err
timeout 600 $B --config 3 --flags 128 > $D/c3_mid.json 2> $D/c3_mid.err
timeout 600 $B --config 4 --l2-fetch 32 > $D/c4_l2f32.json 2> $D/c4_l2f32.err
echo done
