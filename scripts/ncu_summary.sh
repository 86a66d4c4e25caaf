#!/bin/bash
# ncu_summary.sh REP OUT.csv -- per-kernel summary of an `ncu --set full` capture
ncu -i "$1" --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__thread_inst_executed_per_inst_executed.ratio,lts__t_sectors_srcunit_tex_op_atom.sum,launch__grid_size,smsp__average_warp_latency_per_inst_issued.ratio > "$2"
