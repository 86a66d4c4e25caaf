"""A/B helper: cc_spanning_forest time on a config (CUDA events, mean of reps after 2 warm-ups).
usage: sf_ab.py CONFIG [REPS]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import inputs  # noqa: E402
from inputs import gpu as ggen  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

cfg = inputs.BY_INDEX[int(sys.argv[1])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
d_off, d_adj = ggen.config_graph(cfg)
n, m = d_off.numel() - 1, d_adj.numel()
edges = torch.empty((n, 2), dtype=torch.int32, device="cuda")
num = torch.zeros(1, dtype=torch.int64, device="cuda")
lab = torch.empty(n, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for with_lab in (False, True):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cc.cc_spanning_forest(d_off, d_adj, n, m, edges, num, lab if with_lab else None, cc.make_opts())
        e1.record()
        e1.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    print(cfg.name, "labels" if with_lab else "no-labels", round(sum(ts) / len(ts), 4), "ms", int(num.item()))
