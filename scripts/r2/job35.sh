# ncu of the C3 link: refill kernel (flag LINK_REFILL) and k_link_pending with kLB=2
D=gpurun_out/j35; mkdir -p $D
P="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $P --flags 262144 > $D/plain_refill.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_refill" --launch-skip 4 -c 1 -o $D/c3_refill $P --flags 262144 > $D/ncu_refill.log 2>&1
CC_LIBCC_PATH=build/var/libcc_lb2.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_pending" --launch-skip 4 -c 1 -o $D/c3_lb2 $P > $D/ncu_lb2.log 2>&1
echo done
