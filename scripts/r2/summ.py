"""Summarise bench JSON lines: python scripts/r2/summ.py FILES..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAIL", e)
        continue
    k = d.get("kernels", {})
    fin = d.get("finish", {})
    print(f.split("/")[-1], round(d["ms_per_step"], 4), " ".join(f"{x[2:10]}={k[x]['ms']:.4f}" for x in k),
          "fin", fin.get("ms"), "frac8", fin.get("frac_of_8TBs"), "tiles", d.get("counters", {}).get("h6_tiles"))
