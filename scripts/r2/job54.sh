D=gpurun_out/j54; mkdir -p $D
P="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
CC_LIBCC_PATH=build/var/libcc_sp.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_" -c 60 --csv --log-file $D/launches.csv $P > $D/ncu.log 2>&1
echo done
