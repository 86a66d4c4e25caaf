set -x
timeout 900 python scripts/probe/fuzz.py 600 31 > gpurun_out/fuzz_r2_c.txt 2>&1; tail -n 2 gpurun_out/fuzz_r2_c.txt
timeout 900 python scripts/probe/fuzz.py 600 32 > gpurun_out/fuzz_r2_d.txt 2>&1; tail -n 2 gpurun_out/fuzz_r2_d.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/torchrun_n1.json 2> gpurun_out/torchrun_n1.err; tail -c 400 gpurun_out/torchrun_n1.json
echo done
