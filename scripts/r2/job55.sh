# where the CRFA / SV rounds go on C4 at k = 0 after the writeMin test + WarpBuf appends (launch list)
mkdir -p gpurun_out/j55
for f in 8192 512; do
P="python bench.py --config 4 --k 0 --flags $f --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $P > gpurun_out/j55/plain_$f.json 2> gpurun_out/j55/plain_$f.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum --clock-control none -k regex:"k_" -c 200 --csv --log-file gpurun_out/j55/launches_$f.csv $P > gpurun_out/j55/ncu_$f.log 2>&1
done
echo done
