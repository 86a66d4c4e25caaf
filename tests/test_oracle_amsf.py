"""Pins for the minimum-spanning-forest oracles (oracle.kruskal, oracle.amsf).

AMSF (NEXT-4): W(F_OPT) <= W(F_APX) <= (1+eps) W(F_OPT).  The
checks below are chosen so that a plausible slip fails one of them:

* Kruskal against brute force (the minimum over EVERY acyclic edge subset of
  size n - c) on small graphs, against closed forms (triangle 1,1,10 -> 2;
  4-cycle 1,2,3,4 -> 6; edgeless -> 0) and against scipy's
  minimum_spanning_tree (a library routine) on random graphs;
* AMSF: the approximation sandwich on 50 seeded ER graphs and on
  RMAT; exactness when all weights are equal (one bucket); the number of
  forest edges in each bucket equals the rank increase of the prefix graphs,
  (n - c(G_<=i)) - (n - c(G_<i)), computed by scipy's connected_components --
  a property of the bucketing alone, not of the order edges are tried in;
  the forest is valid (forest_check); the bucket index of every forest edge
  satisfies b_i <= w < b_(i+1) and the numpy restatement agrees with the C one;
* the weight generator: symmetric, positive, mean ~ 1, and its fixed-order
  log within 1e-11 of numpy's.
"""
import itertools

import numpy as np
import pytest

import oracle
from inputs import gen
from tests.helpers import csr

sp = pytest.importorskip("scipy.sparse")
csgraph = pytest.importorskip("scipy.sparse.csgraph")


def weighted(n, wedges):
    """CSR + aligned weights from (u, v, w) triples (symmetric)."""
    off, adj = csr(n, [(u, v) for u, v, _ in wedges])
    wmap = {}
    for u, v, w in wedges:
        wmap[(u, v)] = wmap[(v, u)] = np.float32(w)
    src = np.repeat(np.arange(n), np.diff(off))
    w = np.array([wmap[(int(a), int(b))] for a, b in zip(src, adj)], dtype=np.float32)
    return off, adj, w


def n_components(off, adj):
    n = off.size - 1
    g = sp.csr_matrix((np.ones(adj.size), adj.astype(np.int64), off), shape=(n, n))
    return csgraph.connected_components(g, directed=False)[0]


def brute_msf(n, edges):
    """min total weight over all acyclic edge subsets of size n - c (tiny graphs)."""
    par = list(range(n))

    def find(x):
        while par[x] != x:
            x = par[x]
        return x
    for u, v, _ in edges:
        a, b = find(u), find(v)
        if a != b:
            par[a] = b
    c = len({find(x) for x in range(n)})
    best = None
    for sub in itertools.combinations(edges, n - c):
        p = list(range(n))

        def f(x):
            while p[x] != x:
                x = p[x]
            return x
        ok = True
        for u, v, _ in sub:
            a, b = f(u), f(v)
            if a == b:
                ok = False
                break
            p[a] = b
        if ok:
            s = sum(float(np.float32(w)) for _, _, w in sub)
            best = s if best is None else min(best, s)
    return best if best is not None else 0.0


# ---------------------------------------------------------------------------
def test_kruskal_closed_forms():
    off, adj, w = weighted(3, [(0, 1, 1), (1, 2, 1), (0, 2, 10)])
    assert oracle.kruskal(off, adj, w)[0] == 2.0
    off, adj, w = weighted(4, [(0, 1, 1), (1, 2, 2), (2, 3, 3), (3, 0, 4)])
    tot, F, Fw = oracle.kruskal(off, adj, w)
    assert tot == 6.0 and F.shape == (3, 2) and sorted(Fw.tolist()) == [1.0, 2.0, 3.0]
    off, adj = csr(5, [])
    assert oracle.kruskal(off, adj, np.zeros(0, np.float32))[0] == 0.0


def test_kruskal_brute_force_small():
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(2, 7))
        pairs = [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < 0.6]
        edges = [(u, v, float(rng.integers(1, 9))) for u, v in pairs]      # ties on purpose
        off, adj, w = weighted(n, edges)
        assert oracle.kruskal(off, adj, w)[0] == pytest.approx(brute_msf(n, edges), abs=1e-9), (n, edges)


def test_kruskal_vs_scipy():
    for seed in range(4):
        off, adj = gen.er(seed=seed + 10, n0=3000, pairs=9000, isolated=7)
        w = gen.exp_weights(off, adj, seed)
        n = off.size - 1
        g = sp.csr_matrix((w.astype(np.float64), adj.astype(np.int64), off), shape=(n, n))
        want = csgraph.minimum_spanning_tree(g).sum()
        tot, F, _ = oracle.kruskal(off, adj, w)
        assert tot == pytest.approx(want, rel=1e-9)
        assert F.shape[0] == n - n_components(off, adj)


# ---------------------------------------------------------------------------
def check_amsf(off, adj, w, eps):
    n = off.size - 1
    wopt = oracle.kruskal(off, adj, w)[0]
    r = oracle.amsf(off, adj, w, eps)
    assert wopt <= r["total"] * (1 + 1e-12) and r["total"] <= (1 + eps) * wopt * (1 + 1e-12)
    c = n_components(off, adj)
    assert oracle.forest_check(off, adj, c, r["pairs"])[0] == 0
    if adj.size:
        b = oracle.amsf_bounds(w.min(), w.max(), eps)
        assert len(b) - 1 == r["nbuckets"]
        assert np.array_equal(oracle.amsf_bucket(r["weights"], b), r["buckets"])
        bi = r["buckets"]
        assert np.all(b[bi] <= r["weights"].astype(np.float64))
        assert np.all(r["weights"].astype(np.float64) < b[bi + 1])
        # rank increase of the prefix graphs, bucket by bucket (scipy)
        eb = oracle.amsf_bucket(w, b)
        prev = n
        for i in range(r["nbuckets"]):
            keep = eb <= i
            src = np.repeat(np.arange(n), np.diff(off))[keep]
            g = sp.csr_matrix((np.ones(int(keep.sum())), (src, adj[keep].astype(np.int64))), shape=(n, n))
            ci = csgraph.connected_components(g, directed=False)[0]
            assert int(np.sum(bi == i)) == prev - ci, i
            prev = ci
    return r, wopt


def test_amsf_closed_forms():
    off, adj, w = weighted(3, [(0, 1, 1), (1, 2, 1), (0, 2, 10)])
    r, _ = check_amsf(off, adj, w, 0.25)
    assert r["total"] == 2.0
    off, adj = gen.er(seed=3, n0=500, pairs=2000, isolated=3)
    w = np.full(adj.size, 3.5, dtype=np.float32)                        # one bucket: exact
    r, wopt = check_amsf(off, adj, w, 0.25)
    assert r["nbuckets"] == 1 and r["total"] == wopt
    # boundaries at W_min = 1, eps = 1: [1,2) [2,4); w = 2 lies in bucket 1 (half-open
    # on the right), where CSR order tries (0,2) w=3.9 before (1,2) w=2: total 4.9;
    # a bucket rule closed on the right would give the optimum 3
    off, adj, w = weighted(3, [(0, 1, 1.0), (1, 2, 2.0), (0, 2, 3.9)])
    r, wopt = check_amsf(off, adj, w, 1.0)
    assert wopt == 3.0 and r["total"] == pytest.approx(4.9, abs=1e-6) and r["buckets"].tolist() == [0, 1]
    # self-loops are entries of the input: a loop of weight 0.001 sets W_min (reading R25),
    # eps = 1 gives b_i = 0.001 * 2^i, so w = 1.0 is in bucket 9 ([0.512, 1.024)), w = 1.5
    # in bucket 10 and nb = 11 (b_11 = 2.048 > W_max); a loop never joins the forest
    off, adj = csr(3, [(0, 1), (1, 2), (2, 2)], keep_loops=True)
    w = np.array([1.0, 1.0, 1.5, 1.5, 0.001], dtype=np.float32)        # CSR: 0:[1] 1:[0,2] 2:[1,2]
    r = oracle.amsf(off, adj, w, 1.0)
    assert r["nbuckets"] == 11 and r["buckets"].tolist() == [9, 10] and r["total"] == 2.5
    off, adj = csr(4, [])
    r = oracle.amsf(off, adj, np.zeros(0, np.float32), 0.25)
    assert r["total"] == 0.0 and r["pairs"].shape == (0, 2)
    with pytest.raises(ValueError):
        oracle.amsf(*weighted(2, [(0, 1, 0.0)]), 0.25)                   # weights must be > 0
    with pytest.raises(ValueError):
        oracle.amsf(*weighted(2, [(0, 1, 1.0)]), 0.0)                    # eps must be > 0


def test_amsf_sandwich_er_50_seeds():
    """ER(n=1000, avg deg 8), Exp(1), eps = 0.25, 50 seeds."""
    for seed in range(50):
        off, adj = gen.er(seed=100 + seed, n0=1000, pairs=4000, isolated=0)
        check_amsf(off, adj, gen.exp_weights(off, adj, seed), 0.25)


@pytest.mark.parametrize("eps", [0.05, 0.25, 1.0])
def test_amsf_sandwich_rmat_and_grid(eps):
    for off, adj in (gen.rmat(seed=5, scale=11), gen.grid(seed=2, rows=40, cols=33)):
        check_amsf(off, adj, gen.exp_weights(off, adj, 9), eps)


def test_exp_weights_generator():
    off, adj = gen.rmat(seed=4, scale=12)
    w = gen.exp_weights(off, adj, 4)
    n = off.size - 1
    src = np.repeat(np.arange(n), np.diff(off))
    key = {(int(a), int(b)): float(x) for a, b, x in zip(src, adj, w)}
    assert all(key[(b, a)] == x for (a, b), x in key.items())              # symmetric
    assert w.min() > 0 and abs(float(w.mean()) - 1.0) < 0.05
    x = np.concatenate([np.random.default_rng(1).random(10000) * 0.999 + 1e-12, 1 - np.arange(1, 50) * 2.0 ** -53])
    assert np.max(np.abs(gen.neg_ln_fixed(x) + np.log(x)) / np.abs(np.log(x))) < 1e-11


def test_amsf_self_loops_keep_the_guarantee():
    """Reading R25 counts self-loop entries in W_min / W_max.  Pin it to what the paper fixes
    rather than to itself: with loops lighter and heavier than every real edge (so the
    reading moves every bucket boundary), the result is still a valid spanning forest of input
    edges whose per-bucket sizes are the rank increases of the prefix graphs (scipy), inside
    the (1+eps) sandwich around Kruskal -- and a loop never enters the forest."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        off0, adj0 = gen.er(seed=200 + trial, n0=300, pairs=900, isolated=2)
        n = off0.size - 1
        src = np.repeat(np.arange(n), np.diff(off0))
        pairs = [(int(a), int(b)) for a, b in zip(src, adj0) if a < b]
        loops = rng.choice(n, size=12, replace=False)
        off, adj = csr(n, pairs + [(int(x), int(x)) for x in loops], keep_loops=True)
        w = gen.exp_weights(off, adj, trial)
        src = np.repeat(np.arange(n), np.diff(off))
        is_loop = src == adj
        w[is_loop] = np.where(rng.random(int(is_loop.sum())) < 0.5, w.min() * 1e-3, w.max() * 7).astype(np.float32)
        for eps in (0.25, 1.0):
            r, wopt = check_amsf(off, adj, w, eps)
            P = r["pairs"]
            assert not np.any(P[:, 0] == P[:, 1])
