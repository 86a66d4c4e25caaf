# k_finish_proc few-candidates split: static GPU tests, then A/B (cur = split, nosplit = before)
D=gpurun_out/${1:-split}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_static.py tests/test_gpu_full.py -m gpu -x -q -k "not amsf" > $D/pytest.log 2>&1; tail -n 3 $D/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10"
for c in 3 4 1 2; do for rep in 1 2; do for v in cur nosplit; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 $B --config $c > $D/c${c}_${v}_$rep.json 2> $D/c${c}_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c${c}_${v}_$rep.json'));print('c$c $v', d['ms_per_step'], d['finish']['t_fin_ms'], {k:x['ms'] for k,x in d['kernels'].items() if 'finish' in k})"
done; done; done
echo done
