# where AMSF-NF-S's C4 call goes: per-kernel launch list (ncu) of one cc_amsf call
D=gpurun_out/j49; mkdir -p $D
timeout 600 python scripts/probe/amsf_once.py 4 0 3 > $D/plain.txt 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_amsf|k_forest|k_" -c 2000 --csv --log-file $D/launches.csv python scripts/probe/amsf_once.py 4 0 1 > $D/ncu.log 2>&1
echo done
