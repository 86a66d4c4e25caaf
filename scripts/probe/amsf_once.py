"""Probe: one cc_amsf call on a BASELINE config with the seeded Exp(1) weights (for ncu)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import inputs  # noqa: E402
from inputs import gpu as ggen  # noqa: E402
import paper_2008_03909_b200 as pkg  # noqa: E402

cfg = inputs.BY_INDEX[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
d_off, d_adj = ggen.config_graph(cfg)
d_w = ggen.exp_weights(d_off, d_adj, cfg.seed)
torch.cuda.synchronize()
E, W, tot = pkg.amsf(d_off, d_adj, d_w, 0.25, flags=flags)
torch.cuda.synchronize()
print(cfg.name, E.shape[0], tot)
