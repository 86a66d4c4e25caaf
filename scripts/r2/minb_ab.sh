# k_sample_init register cap: cur (3 blocks/SM, 80 regs, 8 B spill) vs minb2 (2 blocks/SM, no spill)
D=gpurun_out/${1:-minb}; mkdir -p $D
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 4 3; do for rep in 1 2; do for v in cur minb2; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c${c}_${v}_$rep.json'));print('c$c $v', d['ms_per_step'], d['kernels']['k_sample_init']['ms'])"
done; done; done
echo done
