# A/B: L2 persistence window over P (env CC_L2_PERSIST = fraction of the max set-aside)
D=gpurun_out/${1:-l2p}; mkdir -p $D
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 3 4 2; do for rep in 1 2; do for v in 0 1.0 0.5; do
  CC_L2_PERSIST=$v timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c${c}_${v}_$rep.json'));print('c$c v$v', d['ms_per_step'], {k:v['ms'] for k,v in d['kernels'].items()}, d['parity'])"
done; done; done
grep -h CC_L2 $D/*.err | sort | uniq -c
echo done
