"""Probe: per-kernel times (cc_opts.marks) of cc_labels with the CSR and labels in pinned
host memory (the zero-copy e2e path) on a config."""
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
h_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
h_adj = torch.empty(m, dtype=torch.int32, pin_memory=True)
h_lab = torch.empty(n, dtype=torch.int32, pin_memory=True)
h_off.copy_(d_off)
h_adj.copy_(d_adj)
del d_off, d_adj
torch.cuda.empty_cache()
s = torch.cuda.current_stream()
acc = None
for rep in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(cc.NUM_MARKS)]
    for e in ev:
        e.record(s)
    torch.cuda.synchronize()
    cc.cc_labels(h_off, h_adj, n, m, h_lab, cc.make_opts(marks=[e.cuda_event for e in ev]), s)
    torch.cuda.synchronize()
    t = [ev[j - 1].elapsed_time(ev[j]) for j in range(1, cc.NUM_MARKS)]
    if rep >= 1:
        acc = t if acc is None else [a + b for a, b in zip(acc, t)]
print({cc.MARK_NAMES[j]: round(acc[j - 1] / 3, 3) for j in range(1, cc.NUM_MARKS)}, "total", round(sum(acc) / 3, 2))
