"""Merge into profiles/ncu_traffic.json the DRAM read+write bytes per launch of one
`ncu --set full` capture, keyed by WORKLOAD then by bench.py mark name:
    python scripts/ncu_traffic.py REP WORKLOAD [NOTE]
bench.py reads only the entry of the workload it runs (None when absent)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, workload = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# the bench marks: k_link_pending is the span of whichever k-out link kernel ran; the final
# compress is k_relabel (partial H6) or the second k_compress (full H6)
alias = {"k_link_refill": "k_link_pending", "k_link_pending": "k_link_pending", "k_relabel": "k_compress_H6"}
res = {}
ncompress = 0
for r in rows[2:]:
    name = r[ki].replace("void ", "").split("(")[0].split("<")[0].split("::")[-1]
    key = alias.get(name, name)
    if name == "k_compress":                      # first: the (gated) mid compress, second: H6
        key = "k_compress_mid" if ncompress == 0 else "k_compress_H6"
        ncompress += 1
    b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
    if key not in res:
        res[key] = int(b)
res["_source"] = f"{os.path.basename(rep)}: ncu --set full --clock-control none, first launch of each kernel; " \
                 f"dram__bytes_read.sum + dram__bytes_write.sum per launch. {note}".strip()
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
try:
    allw = json.load(open(path))
    if "_source" in allw:                         # the round-1 flat layout (C4 only): re-key it
        allw = {"C4-rmat-27(r1 code)": allw}
except Exception:
    allw = {}
allw[workload] = res
json.dump(allw, open(path, "w"), indent=1)
print(json.dumps(res))
