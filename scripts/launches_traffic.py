"""From an ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`) of `bench.py --config C ...`, take one production cc_labels call
(the CALL-th run of the labels kernels, counted by its k_sample_init<..., SF=false, ...>
launch), print its per-kernel times / shares / DRAM bytes, and merge the DRAM read + write
bytes per launch into profiles/ncu_traffic.json under WORKLOAD, keyed by bench.py mark names
(the same aliases as scripts/ncu_traffic.py):
    python scripts/launches_traffic.py LAUNCHES.csv WORKLOAD [CALL] [--no-write]"""
import collections
import csv
import json
import os
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
path_csv, workload = args[0], args[1]
call_no = int(args[2]) if len(args) > 2 else 3
write = "--no-write" not in sys.argv

rows = [r for r in csv.reader(open(path_csv)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(int(r[ii]), {"full": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))


def short(full):
    return full.replace("void ", "").split("(")[0].split("<")[0].split("::")[-1]


# call starts: k_sample_init launches of the labels path (template arg SF = false)
starts = [i for i, d in per.items()
          if short(d["full"]) == "k_sample_init" and "<" in d["full"] and d["full"].split("<")[1].split(",")[1].strip() in ("0", "false")]
if len(starts) < call_no:
    sys.exit(f"only {len(starts)} labels calls in {path_csv}")
ids = list(per.keys())
a = ids.index(starts[call_no - 1])
b = ids.index(starts[call_no]) if call_no < len(starts) else len(ids)
call = []
for i in ids[a:b]:
    name = short(per[i]["full"])
    if not name.startswith("k_"):
        break
    call.append((name, per[i]))
    if name in ("k_relabel",) or (name == "k_compress" and sum(1 for n, _ in call if n == "k_compress") == 2):
        break
tot = sum(d.get("gpu__time_duration.sum", 0.0) for _, d in call)
print(f"{workload}: call {call_no}: total {tot / 1e6:.4f} ms")
alias = {"k_link_refill": "k_link_pending", "k_link_pending": "k_link_pending", "k_relabel": "k_compress_H6",
         "k_relabel_decide": "k_compress_H6"}
res, ncomp = {}, 0
for name, d in call:
    t = d.get("gpu__time_duration.sum", 0.0)
    byts = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    print(f"  {name:18s} {t / 1e6:8.4f} ms  {100 * t / tot:5.1f} %  {byts / 1e9:8.4f} GB")
    key = alias.get(name, name)
    if name == "k_compress":
        key = "k_compress_mid" if ncomp == 0 else "k_compress_H6"
        ncomp += 1
    if name.startswith("k_relabel"):              # the partial H6 is two kernels: their sum
        res[key] = res.get(key, 0) + int(byts)
    elif key not in res or byts > res[key]:       # the gated-out link kernel exits at once: the one that ran
        res[key] = int(byts)
res["_source"] = (f"{os.path.basename(path_csv)} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  f"dram__bytes_write.sum --clock-control none; cold cache per launch), labels call {call_no}; "
                  f"k_compress_H6 = k_relabel_decide + k_relabel when the partial H6 ran")
if write:
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    allw = json.load(open(out)) if os.path.exists(out) else {}
    allw[workload] = res
    json.dump(allw, open(out, "w"), indent=1)
