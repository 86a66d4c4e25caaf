# k_relabel_decide grid (one tile per lane) vs the resident grid: static GPU tests, then A/B
D=gpurun_out/${1:-decide}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_static.py -m gpu -x -q > $D/pytest.log 2>&1; tail -n 3 $D/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 20"
for c in 4 3 1; do for rep in 1 2 3; do for v in cur wide; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c${c}_${v}_$rep.json'));print('c$c $v', d['ms_per_step'], d['finish']['t_fin_ms'], d['kernels']['k_compress_H6']['ms'])"
done; done; done
echo done
