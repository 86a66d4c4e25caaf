set -x
timeout 900 python scripts/probe/fuzz.py 600 21 > gpurun_out/fuzz_r2_a.txt 2>&1; tail -2 gpurun_out/fuzz_r2_a.txt
timeout 900 python scripts/probe/fuzz.py 600 22 > gpurun_out/fuzz_r2_b.txt 2>&1; tail -2 gpurun_out/fuzz_r2_b.txt
timeout 300 python scripts/probe/shapes.py > gpurun_out/shapes_r2.txt 2>&1; tail -5 gpurun_out/shapes_r2.txt
echo done
