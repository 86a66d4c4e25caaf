"""Probe: cc_labels time on adversarial shapes (long chains, stars, full grids), checked vs the oracle."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from inputs import gen  # noqa: E402
import paper_2008_03909_b200 as pkg  # noqa: E402


def csr_pairs(n, u, v):
    return oracle.csr_from_pairs(n, np.stack([u, v], 1))


def shapes(n):
    ids = np.arange(n - 1, dtype=np.uint64)
    yield "path_ascending", csr_pairs(n, ids, ids + 1)
    perm = np.random.default_rng(1).permutation(n).astype(np.uint64)
    yield "path_permuted", csr_pairs(n, perm[:-1], perm[1:])
    yield "star_center0", csr_pairs(n, np.zeros(n - 1, np.uint64), ids + 1)
    yield "star_center_last", csr_pairs(n, np.full(n - 1, n - 1, np.uint64), ids)
    side = int(np.sqrt(n))
    yield "grid_full", gen.grid(seed=1, rows=side, cols=side, p32=1 << 32)
    yield "two_paths_interleaved", csr_pairs(n, ids[:-1], ids[:-1] + 2)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
for name, (off, adj) in shapes(n):
    d_off = torch.from_numpy(off).cuda()
    d_adj = torch.from_numpy(adj.view(np.int32)).cuda()
    t0 = time.time()
    want = oracle.cc_bfs(off, adj)
    t_or = time.time() - t0
    for k in (2, 0):
        lab = pkg.connected_components(d_off, d_adj, k=k)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pkg.connected_components(d_off, d_adj, k=k, out=lab)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = np.array_equal(lab.cpu().numpy().view(np.uint32), want)
        print(f"{name:24s} k={k} n={off.size - 1:9d} m={adj.size:10d} gpu {min(ts):8.3f} ms  bit-exact={ok}"
              f"  (oracle {t_or:.1f}s)", flush=True)

# incremental: a path inserted in id order (one batch, then 16 batches), then 2^20 queries
inc_n = n
ids = torch.arange(inc_n - 1, device="cuda", dtype=torch.int64)
path = torch.stack([ids, ids + 1], 1).to(torch.int32).contiguous()
g = torch.Generator(device="cuda").manual_seed(1)
qs = torch.randint(0, inc_n, (1 << 20, 2), device="cuda", dtype=torch.int64, generator=g).to(torch.int32)
for nb in (1, 16):
    for flags in (0, pkg.cc.FLAG_FIND_SPLIT):
        inc = pkg.IncrementalCC(inc_n, flags=flags)
        empty = torch.empty((0, 2), dtype=torch.int32, device="cuda")
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        e0.record()
        step = (inc_n - 1 + nb - 1) // nb
        for b in range(nb):
            inc.batch(path[b * step:(b + 1) * step].contiguous(), empty)
        e1.record()
        ans = inc.batch(empty, qs)
        e2.record()
        e2.synchronize()
        print(f"incr path n={inc_n} batches={nb} flags={flags}: inserts {e0.elapsed_time(e1):9.3f} ms, "
              f"2^20 queries {e1.elapsed_time(e2):9.3f} ms, all true={bool(ans.all().item())}", flush=True)
        inc.close()
