"""The north_star's three ncu counters per kernel (achieved DRAM GB/s, L2 sector hit rate,
L2 atomic sectors / s) from `ncu --page raw --csv` exports that carry gpu__time_duration.sum,
dram__bytes_{read,write}.sum, lts__t_sector_hit_rate.pct and lts__t_sectors_srcunit_tex_op_atom.sum:
    python scripts/ncu_counters.py profiles/r2_ncu_full_c4.csv [more.csv ...]"""
import csv
import sys

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1.0, "us": 1e-3, "usecond": 1e-3,
         "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6}
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h, u = rows[0], rows[1]
    ix = {c: h.index(c) for c in h}

    def val(r, c):
        return float(r[ix[c]].replace(",", "")) * SCALE.get(u[ix[c]], 1.0)

    print(f"{f}:")
    print(f"  {'kernel':28s} {'ms':>8s} {'DRAM GB':>8s} {'GB/s':>7s} {'L2 hit':>7s} {'atom sectors':>13s} {'atom G/s':>9s}")
    for r in rows[2:]:
        name = r[ix["Kernel Name"]].replace("void ", "").split("(")[0].split("::")[-1][:28]
        ms = val(r, "gpu__time_duration.sum")
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        atom = float(r[ix["lts__t_sectors_srcunit_tex_op_atom.sum"]].replace(",", ""))
        hit = float(r[ix["lts__t_sector_hit_rate.pct"]])
        print(f"  {name:28s} {ms:8.4f} {dram / 1e9:8.3f} {dram / ms / 1e6:7.0f} {hit:6.1f}% {atom / 1e6:11.2f} M "
              f"{atom / ms / 1e6:9.2f}")
