# last code: the NEXT-2 sweep again (its multi-batch rows use the pre-wait reads now), and the
# torchrun launch path of bench.py at N = 1 (NCCL init, barrier, max-over-ranks)
D=gpurun_out/${1:-extras}; mkdir -p $D
timeout 1200 python bench.py --incr-sweep > $D/incr_sweep.json 2> $D/incr_sweep.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $D/torchrun_n1.json 2> $D/torchrun_n1.err
tail -c 400 $D/torchrun_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 > $D/torchrun_ref_n1.json 2> $D/torchrun_ref_n1.err
tail -c 300 $D/torchrun_ref_n1.json
echo done
