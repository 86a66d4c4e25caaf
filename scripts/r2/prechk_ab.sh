# link hook pre-check (fresh L2 read before the CAS): cur vs prechk on C1, C3, C4, C2
D=gpurun_out/${1:-prechk}; mkdir -p $D
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 1 3 4 2; do for rep in 1 2; do for v in cur prechk; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c${c}_${v}_$rep.json'));print('c$c $v', d['ms_per_step'], d['kernels']['k_link_pending']['ms'], d['counters']['cas_failures'], d['counters']['link_steps'])"
done; done; done
echo done
