for c in 1 2 3; do timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 python bench.py --config 4 --k 0 > gpurun_out/bench_c4_k0.json 2> gpurun_out/bench_c4_k0.err
