"""Per cc_labels call breakdown of an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv): every run of libcc kernels from
k_sample_init to the final compress (k_relabel / second k_compress), with each kernel's
time, share of the call and DRAM bytes.   usage: ncu_step.py LAUNCHES.csv [CALL_INDEX ...]"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(int(r[ii]), {})
    d[r[mi]] = float(r[vi].replace(",", ""))
    d["name"] = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
calls, cur = [], None
# a call ends with its final compress: k_relabel (partial H6, after k_relabel_decide)
for i, d in per.items():
    if d["name"] == "k_sample_init":
        cur = []
        calls.append(cur)
    if cur is not None:
        cur.append(d)
        if d["name"] in ("k_relabel",):
            cur = None
want = [int(x) for x in sys.argv[2:] if x != "--json"] or list(range(len(calls)))
out = []
for c in want:
    ks = calls[c]
    tot = sum(k["gpu__time_duration.sum"] for k in ks)
    rows_c = [{"kernel": k["name"], "ms": round(k["gpu__time_duration.sum"] / 1e6, 5),
               "share": round(k["gpu__time_duration.sum"] / tot, 4),
               "dram_bytes": int(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0))} for k in ks]
    out.append({"call": c, "total_ms": round(tot / 1e6, 5), "kernels": rows_c})
    print(f"call {c}: total {tot / 1e6:.4f} ms")
    for r in rows_c:
        print(f"  {r['kernel']:16s} {r['ms']:9.4f} ms  {100 * r['share']:5.1f} %  {r['dram_bytes'] / 1e9:7.3f} GB")
if "--json" in sys.argv:
    print(json.dumps(out))
