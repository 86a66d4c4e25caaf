"""Build profiles/r2_next3_sv_crfa.json from bench lines named c{C}_k{K}_f{F}.json in a directory
(python bench.py --config C --k K --flags F --steps 3 --warmup 3 --no-e2e --no-cpu-baseline)."""
import json
import pathlib
import sys

src = pathlib.Path(sys.argv[1])
names = {0: "UF-Rem-CAS + SplitAtomicOne (default)", 512: "Shiloach-Vishkin (CC_FLAG_FINISH_SV)",
         8192: "Liu-Tarjan CRFA (CC_FLAG_FINISH_CRFA)"}
rows = []
for c in (2, 4):
    for k in (0, 2):
        base = None
        for f in (0, 512, 8192):
            d = json.loads((src / f"c{c}_k{k}_f{f}.json").read_text().strip().splitlines()[-1])
            fin = d["finish"]["t_fin_ms"]
            if f == 0:
                base = d["ms_per_step"]
            rows.append({"workload": d["config"]["workload"], "kout_k": k, "finish": names[f], "flags": f,
                         "ms_per_step": round(d["ms_per_step"], 5), "finish_phase_ms": round(fin, 5),
                         "rounds": d["counters"]["sv_rounds"] or None, "GTEPS": round(d["value"], 4),
                         "slowdown_vs_uf": round(d["ms_per_step"] / base, 2),
                         "spanning_forest_ms": round(d.get("spanning_forest", {}).get("ms", 0.0), 3)})
out = {"study": "NEXT-3: second finish family vs UF-Rem-CAS (SURVEY 8(f) NEXT-3; paper: SV 2.98-7.62x, "
                "LT 2.64-10.2x slower than UF-Rem-CAS on 72 cores, P:1296-1305)",
       "source": f"{src}: python bench.py --config {{2,4}} --k {{0,2}} --flags {{0,512,8192}} --steps 3 --warmup 3 "
                 "--no-e2e --no-cpu-baseline, one B200",
       "rows": rows}
print(json.dumps(out, indent=1))
