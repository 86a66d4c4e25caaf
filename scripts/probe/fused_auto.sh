# auto-fuse A/B: default library (auto), NO_FUSE (131072), and the evict-first build
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
for c in 3 1 2 4; do
  for run in "def 0" "def 131072" "slef 0"; do
    set -- $run
    lib=paper_2008_03909_b200/libcc.so; [ $1 = slef ] && lib=build/var/libcc_slef.so
    CC_LIBCC_PATH=$lib timeout 300 python bench.py --config $c --steps 20 --warmup 3 --flags $2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/fa.json
    python -c "
import json; d=json.load(open('gpurun_out/fa.json'))
print('C$c', '$1', $2, d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['kernels'].items()}, d['counters']['fused_link'], d['roofline'].get('random_access_view',{}).get('frac_of_random_gather_rate'))"
  done
done
