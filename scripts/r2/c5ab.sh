# C5 A/B of build variants + ncu launch list of the C5 stream: bash scripts/r2/c5ab.sh OUT "cur v1 ..."
D=gpurun_out/$1; mkdir -p $D
B="python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 5 --warmup 3"
for rep in 1 2; do
  for v in $2; do
    if [ $v = cur ]; then L=""; else L="CC_LIBCC_PATH=build/var/libcc_$v.so"; fi
    env $L timeout 600 $B > $D/c5_${v}_$rep.json 2> $D/c5_${v}_$rep.err
    python -c "import json,sys;d=json.load(open('$D/c5_${v}_$rep.json'));print('$v',d['value'],d['ms_per_step'],d['roofline']['random_access_view'])"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $D/launches_c5.csv python bench.py --config 5 --no-e2e --no-cpu-baseline --steps 1 --warmup 1 > $D/ncu_c5.log 2>&1
echo done
