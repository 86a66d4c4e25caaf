"""Probe: cc_amsf on a BASELINE config with the seeded Exp(1) weights (for ncu / A-B).
usage: amsf_once.py [config=3] [flags=0] [reps=1] -- prints ms per call (CUDA events) and counters."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import inputs  # noqa: E402
from inputs import gpu as ggen  # noqa: E402
import paper_2008_03909_b200 as pkg  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

cfg = inputs.BY_INDEX[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
d_off, d_adj = ggen.config_graph(cfg)
d_w = ggen.exp_weights(d_off, d_adj, cfg.seed)
torch.cuda.synchronize()
ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
E, W, tot = pkg.amsf(d_off, d_adj, d_w, 0.25, flags=flags, counters=ctr)
ts = []
for _ in range(reps - 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pkg.amsf(d_off, d_adj, d_w, 0.25, flags=flags)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
if os.environ.get("DEGSTATS"):
    deg = (d_off[1:] - d_off[:-1])
    m = int(d_off[-1].item())
    for lo, hi in ((0, 0), (1, 32), (33, 256), (257, 4096), (4097, 1 << 40)):
        sel = (deg >= lo) & (deg <= hi)
        print(f"deg {lo}-{hi}: vertices {int(sel.sum().item())} entries {int(deg[sel].sum().item()) / m:.3f}")
print(cfg.name, "forest", E.shape[0], "W", tot, "ms", [round(t, 2) for t in ts],
      {k: v for k, v in c.items() if k.startswith("amsf")})
