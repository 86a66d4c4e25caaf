"""Keep the columns the profiles cite from an `ncu -i REP --page raw --csv` export:
    python scripts/ncu_select.py RAW.csv OUT.csv"""
import csv
import sys

KEEP = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__thread_inst_executed_per_inst_executed.ratio"]
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
cols = list(range(11)) + [h.index(c) for c in KEEP if c in h]
with open(sys.argv[2], "w", newline="") as f:
    w = csv.writer(f, quoting=csv.QUOTE_ALL)
    for r in rows:
        w.writerow([r[i] for i in cols])
