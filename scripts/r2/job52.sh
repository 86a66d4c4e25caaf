# feasibility: k_link_pending in N passes over the pending list, pass b linking only v in the b-th range of ids
mkdir -p gpurun_out/j52
bash scripts/r2/ab.sh j52 "cur vp2 vp4 vp8" "4 3"
