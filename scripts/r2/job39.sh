mkdir -p gpurun_out/j39
bash scripts/r2/ab.sh j39 "cur d1 d2 d3" "3 4"
