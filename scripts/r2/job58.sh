# final SV / CRFA copy: full-size C4 parity (k=0 SV / CRFA) and the NEXT-3 table
mkdir -p gpurun_out/j58
timeout 1400 python -m pytest tests/test_gpu_full.py -x -q -k "no_sampling" > gpurun_out/j58/full.log 2>&1; echo "rc=$?" >> gpurun_out/j58/full.log
sed -i 's#^D=gpurun_out/j44#D=gpurun_out/j58#' scripts/r2/job44.sh
bash scripts/r2/job44.sh
