# the fuzz campaign on the final round-2 code (after the pieced SV/CRFA edge copy): two seeds x 600 s
D=gpurun_out/${1:-fuzz}; mkdir -p $D
timeout 700 python scripts/probe/fuzz.py 600 101 > $D/fuzz_101.txt 2>&1; echo "rc=$?" >> $D/fuzz_101.txt
timeout 700 python scripts/probe/fuzz.py 600 202 > $D/fuzz_202.txt 2>&1; echo "rc=$?" >> $D/fuzz_202.txt
for f in $D/fuzz_*.txt; do tail -n 2 $f; done
