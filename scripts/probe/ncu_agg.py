"""Aggregate an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
launch list per kernel name: launches, total time, share, DRAM bytes, DRAM GB/s.
usage: ncu_agg.py LAUNCHES.csv [TOP]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    per[r[ii]]["name"] = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for v in per.values():
    a = agg[v["name"]]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0.0)
    a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else None
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k:22s} n={a[0]:4d} ms={a[1] / 1e6:8.3f} share={a[1] / tot:.3f} dram={a[2] / 1e9:8.2f} GB "
          f"GB/s={a[2] / max(a[1], 1e-9):8.1f}")
print(f"total ms={tot / 1e6:.3f}")
