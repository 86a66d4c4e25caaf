"""Fuzz: random graphs (ER / RMAT / grid / stars / paths / cliques, random id
permutations, duplicates and self-loops) x random options through cc_labels,
cc_spanning_forest, cc_amsf and cc_incr_batch, every result checked against the
oracle.  Usage: fuzz.py SECONDS SEED.  Prints a summary; exits 1 on a mismatch."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from inputs import gen  # noqa: E402
import paper_2008_03909_b200 as pkg  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
FLAGS = [0, cc.FLAG_HALVE, cc.FLAG_UF_ASYNC, cc.FLAG_NO_SKIP, cc.FLAG_NO_MIDCOMPRESS, cc.FLAG_MIDCOMPRESS,
         cc.FLAG_NO_DEGSKIP, cc.FLAG_FINISH_SV, cc.FLAG_FINISH_CRFA, cc.FLAG_CONTRACT, cc.FLAG_NO_REFILL, cc.FLAG_FUSED_LINK]


def random_graph():
    kind = rng.integers(0, 7)
    n = int(rng.integers(1, 30000))
    if kind == 0:
        pairs = rng.integers(0, n, (int(rng.integers(0, 3 * n)), 2))
    elif kind == 1:
        s = int(rng.integers(4, 15))
        off, adj = gen.rmat(seed=int(rng.integers(1 << 30)), scale=s)
        return off, adj, f"rmat{s}"
    elif kind == 2:
        r, c = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        off, adj = gen.grid(seed=int(rng.integers(1 << 30)), rows=r, cols=c, p32=int(rng.integers(1 << 31, 1 << 32)))
        return off, adj, f"grid{r}x{c}"
    elif kind == 3:
        k = int(rng.integers(1, 5))
        centres = rng.integers(0, n, k)
        pairs = np.stack([np.repeat(centres, n // k + 1)[:n], rng.permutation(n)], 1)
    elif kind == 4:
        p = rng.permutation(n) if rng.random() < 0.5 else np.arange(n)
        pairs = np.stack([p[:-1], p[1:]], 1) if n > 1 else np.zeros((0, 2), np.int64)
    elif kind == 5:
        b = int(rng.integers(2, 60))
        v = np.arange(n)
        pairs = np.stack([v, (v // b) * b + rng.integers(0, b, n)], 1)
        pairs = pairs[pairs[:, 1] < n]
    else:
        pairs = np.stack([rng.integers(0, n, 4 * n), rng.integers(0, n, 4 * n)], 1)
        pairs = pairs[np.abs(pairs[:, 0] - pairs[:, 1]) < int(rng.integers(1, 50))]
    off, adj = oracle.csr_from_pairs(n, pairs) if len(pairs) else (np.zeros(n + 1, np.int64), np.zeros(0, np.uint32))
    return off, adj, f"kind{kind}_n{n}"


t0 = time.time()
runs = {"labels": 0, "forest": 0, "amsf": 0, "incr": 0}
while time.time() - t0 < secs:
    off, adj, name = random_graph()
    n = off.size - 1
    want = oracle.cc_bfs(off, adj)
    d_off = torch.from_numpy(off).cuda()
    d_adj = torch.from_numpy(adj.view(np.int32) if adj.size else np.zeros(0, np.int32)).cuda()
    k = int(rng.choice([0, 1, 2, 2, 2, 3, 5]))
    variant = ["afforest", "hybrid", "pure"][int(rng.integers(0, 3))]
    fl = int(rng.choice(FLAGS)) | int(rng.choice(FLAGS))
    seed = int(rng.integers(1 << 30))
    grid = int(rng.choice([0, 0, 0, 1, 3, 37, 1000, 5000]))      # random launch configuration
    cc.set_grid(grid)
    hooks = {}
    if rng.random() < 0.1 and n:                                  # forced L_max (any vertex or none)
        forced = int(rng.integers(0, n)) if rng.random() < 0.8 else 0xFFFFFFFF
        hooks["lmax_force"] = torch.tensor([np.uint32(forced).view(np.int32)], dtype=torch.int32, device="cuda")
    lab = pkg.connected_components(d_off, d_adj, k=k, variant=variant, seed=seed, flags=fl, **hooks)
    got = lab.cpu().numpy().view(np.uint32)
    if not np.array_equal(got, want):
        print("LABELS MISMATCH", name, k, variant, fl, seed, grid, hooks, np.nonzero(got != want)[0][:5])
        sys.exit(1)
    runs["labels"] += 1
    if rng.random() < 0.5:
        wl = rng.random() < 0.7
        edges, lab2 = pkg.spanning_forest(d_off, d_adj, k=k, variant=variant, seed=seed, flags=fl, with_labels=wl)
        c = int(np.sum(want == np.arange(n)))
        rc, bad = oracle.forest_check(off, adj, c, edges.cpu().numpy().view(np.uint32))
        if rc or (wl and not np.array_equal(lab2.cpu().numpy().view(np.uint32), want)):
            print("FOREST MISMATCH", name, k, variant, fl, seed, oracle.FOREST_ERRORS.get(rc), bad)
            sys.exit(1)
        runs["forest"] += 1
    if adj.size and rng.random() < 0.3:
        w = gen.exp_weights(off, adj, seed)
        eps = float(rng.choice([0.05, 0.25, 1.0]))
        afl = int(rng.choice([0, cc.FLAG_NO_SKIP, cc.FLAG_AMSF_PLAIN, cc.FLAG_AMSF_NO_INDEX, cc.FLAG_HALVE]))
        E, W, tot = pkg.amsf(d_off, d_adj, torch.from_numpy(w).cuda(), eps, flags=afl)
        r = oracle.amsf(off, adj, w, eps)
        b = oracle.amsf_bounds(w.min(), w.max(), eps)
        gh = np.bincount(oracle.amsf_bucket(W.cpu().numpy(), b), minlength=r["nbuckets"])
        c = int(np.sum(want == np.arange(n)))
        rc, bad = oracle.forest_check(off, adj, c, E.cpu().numpy().view(np.uint32))
        if rc or not np.array_equal(gh, np.bincount(r["buckets"], minlength=r["nbuckets"])):
            print("AMSF MISMATCH", name, eps, afl, seed, oracle.FOREST_ERRORS.get(rc))
            os.makedirs("gpurun_out", exist_ok=True)
            np.savez("gpurun_out/fuzz_fail.npz", off=off, adj=adj, w=w, eps=eps, flags=afl,
                     E=E.cpu().numpy(), W=W.cpu().numpy(), gh=gh,
                     wh=np.bincount(r["buckets"], minlength=r["nbuckets"]))
            sys.exit(1)
        runs["amsf"] += 1
    if rng.random() < 0.3 and n > 1:
        ifl = int(rng.choice([0, cc.FLAG_HALVE, cc.FLAG_UF_ASYNC, cc.FLAG_FIND_SPLIT, cc.FLAG_FIND_NAIVE]))
        inc = pkg.IncrementalCC(n, flags=ifl)
        batches = []
        for b in range(int(rng.integers(1, 6))):
            ins = rng.integers(0, n, (int(rng.integers(0, 3 * n)), 2)).astype(np.uint32)
            qs = rng.integers(0, n, (int(rng.integers(0, n)), 2)).astype(np.uint32)
            batches.append((ins, qs))
        wa, _ = oracle.incr_run(n, batches)
        ga = [inc.batch(torch.from_numpy(i.view(np.int32)).cuda(), torch.from_numpy(q.view(np.int32)).cuda()).cpu().numpy()
              for i, q in batches]
        inc.close()
        if not np.array_equal(np.concatenate(ga) if ga else np.zeros(0, np.uint8), wa):
            print("INCR MISMATCH", name, ifl)
            sys.exit(1)
        runs["incr"] += 1
        # the same batches through ONE cc_incr_batches call on device arrays (large batches:
        # the kernels after the first read their pairs before their PDL wait)
        ai = np.concatenate([i for i, _ in batches]).reshape(-1, 2)
        aq = np.concatenate([q for _, q in batches]).reshape(-1, 2)
        h = cc.Incr(n, ifl)
        ans = torch.empty(max(1, aq.shape[0]), dtype=torch.uint8, device="cuda")
        h.batches(np.array([i.shape[0] for i, _ in batches], dtype=np.int64), torch.from_numpy(ai.view(np.int32)).cuda(),
                  np.array([q.shape[0] for _, q in batches], dtype=np.int64), torch.from_numpy(aq.view(np.int32)).cuda(),
                  ans)
        h.close()
        if not np.array_equal(ans.cpu().numpy()[:aq.shape[0]], wa):
            print("INCR BATCHES MISMATCH", name, ifl)
            sys.exit(1)
        runs["incr_batches"] = runs.get("incr_batches", 0) + 1
cc.set_grid(0)
print("fuzz ok", runs, f"{time.time() - t0:.0f}s")
