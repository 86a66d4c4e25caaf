# the fuzz campaign on the last code (incl. the multi-batch call with pre-wait reads): two seeds x 600 s
D=gpurun_out/${1:-fuzz2}; mkdir -p $D
timeout 700 python scripts/probe/fuzz.py 600 505 > $D/fuzz_505.txt 2>&1; echo "rc=$?" >> $D/fuzz_505.txt
timeout 700 python scripts/probe/fuzz.py 600 606 > $D/fuzz_606.txt 2>&1; echo "rc=$?" >> $D/fuzz_606.txt
for f in $D/fuzz_*.txt; do tail -n 2 $f; done
