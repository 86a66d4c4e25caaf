timeout 900 python -m pytest tests/test_gpu_amsf.py -x -q 2>&1 | tail -1
for v in def ${VARS:-old}; do lib=paper_2008_03909_b200/libcc.so; [ $v != def ] && lib=build/var/libcc_$v.so
 for f in 4096 0 16384; do echo "$v flags=$f"; CC_LIBCC_PATH=$lib timeout 300 python scripts/probe/amsf_once.py 3 $f 4 2>&1 | tail -1 | cut -c1-90; done; done
