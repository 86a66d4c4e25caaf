"""Write profiles/ncu_traffic.json (DRAM read+write bytes per launch, keyed by the
bench.py mark names) from an `ncu --set full` capture: python scripts/ncu_traffic.py REP."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# the bench marks: k_link_pending is the span of whichever k-out link kernel ran
alias = {"k_link_refill": "k_link_pending", "k_link_pending": "k_link_pending"}
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
res["_source"] = (f"{rep}: ncu --set full --clock-control none on `python bench.py --steps 2 --warmup 1 --no-e2e "
                  "--no-cpu-baseline` (C4 RMAT-27), first cc_labels call; dram__bytes_read.sum + "
                  "dram__bytes_write.sum per launch")
json.dump(res, open("profiles/ncu_traffic.json", "w"), indent=1)
print(res)
