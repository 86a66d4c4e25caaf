"""Probe: per-kernel times (cc_opts.marks) of cc_labels vs cc_spanning_forest on a config."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import inputs  # noqa: E402
from inputs import gpu as ggen  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

cfg = inputs.BY_INDEX[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
d_off, d_adj = ggen.config_graph(cfg)
n, m = d_off.numel() - 1, d_adj.numel()
lab = torch.empty(n, dtype=torch.int32, device="cuda")
edges = torch.empty((n, 2), dtype=torch.int32, device="cuda")
num = torch.zeros(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for name in ("labels", "forest", "forest+labels"):
    acc = None
    for rep in range(6):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(cc.NUM_MARKS)]
        for e in ev:
            e.record(s)
        torch.cuda.synchronize()
        o = cc.make_opts(marks=[e.cuda_event for e in ev])
        if name == "labels":
            cc.cc_labels(d_off, d_adj, n, m, lab, o, s)
        else:
            cc.cc_spanning_forest(d_off, d_adj, n, m, edges, num, lab if name == "forest+labels" else None, o, s)
        torch.cuda.synchronize()
        t = [ev[j - 1].elapsed_time(ev[j]) for j in range(1, cc.NUM_MARKS)]
        if rep >= 2:
            acc = t if acc is None else [a + b for a, b in zip(acc, t)]
    print(name, {cc.MARK_NAMES[j]: round(acc[j - 1] / 4, 4) for j in range(1, cc.NUM_MARKS)},
          "total", round(sum(acc) / 4, 3), flush=True)
