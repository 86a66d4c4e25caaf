mkdir -p gpurun_out/j38
bash scripts/r2/ab.sh j38 "cur h1" "3 4 1 2"
