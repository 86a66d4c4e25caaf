set -x
timeout 600 python scripts/probe/amsf_once.py 4 0 4 > gpurun_out/occ_main.log 2>&1
for v in rmb5 rmb6; do CC_LIBCC_PATH=$PWD/build/var/libcc_$v.so timeout 600 python scripts/probe/amsf_once.py 4 0 4 > gpurun_out/occ_$v.log 2>&1; done
timeout 600 python scripts/probe/amsf_once.py 3 0 4 > gpurun_out/occ3_main.log 2>&1
for v in rmb5 rmb6; do CC_LIBCC_PATH=$PWD/build/var/libcc_$v.so timeout 600 python scripts/probe/amsf_once.py 3 0 4 > gpurun_out/occ3_$v.log 2>&1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
