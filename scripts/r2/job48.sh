# k_finish: tile loads issued before the dependent ctl->lmax -> P[lmax] reads; A/B vs the previous build
mkdir -p gpurun_out/j48
bash scripts/r2/ab.sh j48 "base cur" "4 3 2"
