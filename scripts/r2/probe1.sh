# round-2 probe 1: baseline C3/C4 lines + ncu of the C3 link kernel (source-level)
set -x
mkdir -p gpurun_out/r2p1
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 $B --config 4 --steps 10 > gpurun_out/r2p1/c4.json 2> gpurun_out/r2p1/c4.err
timeout 600 $B --config 3 --steps 10 > gpurun_out/r2p1/c3.json 2> gpurun_out/r2p1/c3.err
timeout 600 $B --config 2 --steps 10 > gpurun_out/r2p1/c2.json 2> gpurun_out/r2p1/c2.err
timeout 600 $B --config 1 --steps 10 > gpurun_out/r2p1/c1.json 2> gpurun_out/r2p1/c1.err
P="python bench.py --config 3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_link_refill" -c 2 -o gpurun_out/r2p1/c3_link $P > gpurun_out/r2p1/ncu_c3.log 2>&1
echo done
