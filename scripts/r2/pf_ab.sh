# incremental pre-wait prefetch: incremental GPU tests, then C5 A/B (cur = prefetch, nopf = before)
D=gpurun_out/${1:-pf}; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_incr.py tests/test_gpu_full.py -m gpu -x -q -k "incr or Incr" > $D/pytest.log 2>&1; tail -n 3 $D/pytest.log
B="python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 5 --warmup 3"
for rep in 1 2 3; do for v in cur nopf; do
  if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
  env $L timeout 600 $B > $D/c5_${v}_$rep.json 2> $D/c5_${v}_$rep.err
  python -c "import json;d=json.load(open('$D/c5_${v}_$rep.json'));print('$v',d['value'],d['ms_per_step'],d['batch_ms'],d['roofline']['random_access_view']['uniform_random_gather_Gloads_per_s'])"
done; done
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 > $D/c5_full_line.json 2> $D/c5_full_line.err
echo done
