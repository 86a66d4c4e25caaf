# AMSF A/B: default library vs build variants (VARS), C4 timing + ncu per-kernel aggregate
timeout 600 python -m pytest tests/test_gpu_amsf.py -x -q 2>&1 | tail -1
for v in def ${VARS}; do
  lib=paper_2008_03909_b200/libcc.so; [ $v != def ] && lib=build/var/libcc_$v.so
  echo "== $v"
  CC_LIBCC_PATH=$lib timeout 300 python scripts/probe/amsf_once.py ${CFG:-4} 0 3 2>&1 | tail -1
  CC_LIBCC_PATH=$lib timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_amsf|k_forest" --log-file gpurun_out/amsf_$v.csv python scripts/probe/amsf_once.py ${CFG:-4} 0 1 > /dev/null 2>&1
  python scripts/probe/ncu_agg.py gpurun_out/amsf_$v.csv ${TOP:-6}
done
