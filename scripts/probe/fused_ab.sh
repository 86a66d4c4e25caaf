# A/B of the fused sampling+link kernel (CC_FLAG_FUSED_LINK = 65536) vs the default path.
timeout 600 python -m pytest tests/test_gpu_static.py -x -q 2>&1 | tail -2
for c in ${CONFIGS:-4 3 2}; do
  for f in ${FLAGS:-0 65536}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --flags $f --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/ab_c${c}_f${f}.json
    python -c "
import json; d=json.load(open('gpurun_out/ab_c${c}_f${f}.json'))
print('C$c', 'flags $f', d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['kernels'].items()}, 'sf', d['spanning_forest']['ms'], 'steps', d['counters']['link_steps'])"
  done
done
