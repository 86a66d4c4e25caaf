for v in ${VARS:-sl4 sl5}; do for c in ${CONFIGS:-4 3}; do
CC_LIBCC_PATH=build/var/libcc_$v.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --flags 65536 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v.json
python -c "
import json; d=json.load(open('gpurun_out/v.json'))
print('$v C$c', d['ms_per_step'], {k: v['ms'] for k, v in d['kernels'].items()})"
done; done
