# the fuzz campaign on the last code (incl. the multi-batch call with pre-wait reads): two seeds x 500 s
D=gpurun_out/${1:-fuzz2}; mkdir -p $D
timeout 600 python scripts/probe/fuzz.py 500 303 > $D/fuzz_303.txt 2>&1; echo "rc=$?" >> $D/fuzz_303.txt
timeout 600 python scripts/probe/fuzz.py 500 404 > $D/fuzz_404.txt 2>&1; echo "rc=$?" >> $D/fuzz_404.txt
for f in $D/fuzz_*.txt; do tail -n 2 $f; done
