"""GPU parity of cc_amsf (AMSF-NF-S, NEXT-4) vs the CPU oracle.

Several forests are correct, so the comparison is on what is unique:
* the forest is a spanning forest of the input (oracle.forest_check);
* every returned weight is the input weight of its edge;
* the number of forest edges in each weight bucket equals the oracle's --
  bit-exact: both sides take the bucket decision b_i <= w < b_(i+1) on the same
  fp64 boundaries (reading R25), and the per-bucket count is the rank increase
  of the prefix graph, a property of the bucketing alone;
* W(F_OPT) <= W(F) <= (1+eps) W(F_OPT) against Kruskal (fp64 sums, 1e-9 slack);
* the returned total equals the fp64 sum of the returned weights.
Everything goes through the C ABI (libcc.so).
"""
import numpy as np
import pytest

import oracle
from inputs import gen
from tests.helpers import fixtures, to_dev, u32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2008_03909_b200 as pkg  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

OPTS = [
    dict(flags=0),
    dict(flags=cc.FLAG_NO_SKIP),
    dict(flags=cc.FLAG_AMSF_PLAIN),
    dict(flags=cc.FLAG_AMSF_PLAIN | cc.FLAG_NO_SKIP),
    dict(flags=cc.FLAG_HALVE, seed=3),
    dict(flags=cc.FLAG_UF_ASYNC, seed=4),
    dict(flags=cc.FLAG_AMSF_NO_INDEX),
]


def run(off, adj, w, eps, **kw):
    d_off, d_adj = to_dev(off, adj)
    d_w = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).cuda()
    E, W, tot = pkg.amsf(d_off, d_adj, d_w, eps, **kw)
    torch.cuda.synchronize()
    return u32(E).reshape(-1, 2), W.cpu().numpy(), tot


def check(off, adj, w, eps, E, W, tot, want=None, exact_opt=True):
    n = off.size - 1
    lab = oracle.cc_bfs(off, adj)
    c = int(np.sum(lab == np.arange(n)))
    rc, bad = oracle.forest_check(off, adj, c, E)
    assert rc == 0, (oracle.FOREST_ERRORS[rc], bad)
    if E.shape[0]:
        # each weight is its edge's input weight
        for (a, b_), x in zip(E[:200], W[:200]):
            lo, hi = off[a], off[a + 1]
            j = lo + np.searchsorted(adj[lo:hi], b_)
            assert w[j] == x
    assert tot == pytest.approx(float(np.sum(W.astype(np.float64))), rel=1e-12, abs=1e-12)
    if adj.size == 0:
        assert E.shape[0] == 0 and tot == 0.0
        return
    want = oracle.amsf(off, adj, w, eps) if want is None else want
    b = oracle.amsf_bounds(w.min(), w.max(), eps)
    got_hist = np.bincount(oracle.amsf_bucket(W, b), minlength=want["nbuckets"])
    want_hist = np.bincount(want["buckets"], minlength=want["nbuckets"])
    assert np.array_equal(got_hist, want_hist), np.nonzero(got_hist != want_hist)[0][:5]
    if exact_opt:
        wopt = oracle.kruskal(off, adj, w)[0]
        assert wopt * (1 - 1e-9) <= tot <= (1 + eps) * wopt * (1 + 1e-9)


def graphs():
    G = [(name, off, adj) for name, off, adj in fixtures()]
    G.append(("er", *gen.er(seed=3, n0=5000, pairs=6000, isolated=37)))
    G.append(("grid", *gen.grid(seed=5, rows=67, cols=131)))
    G.append(("rmat10", *gen.rmat(seed=6, scale=10)))
    G.append(("rmat13_unperm", *gen.rmat(seed=7, scale=13, permuted=False)))
    return G


@pytest.mark.parametrize("opt", OPTS, ids=lambda o: f"f{o['flags']}")
def test_amsf_small(opt):
    for name, off, adj in graphs():
        w = gen.exp_weights(off, adj, 17)
        E, W, tot = run(off, adj, w, 0.25, **opt)
        check(off, adj, w, 0.25, E, W, tot)


@pytest.mark.parametrize("eps", [0.002, 0.01, 0.1, 1.0, 4.0])
def test_amsf_eps(eps):
    off, adj = gen.rmat(seed=8, scale=12)
    w = gen.exp_weights(off, adj, 8)
    for opt in (OPTS[0], OPTS[2]):
        check(off, adj, w, eps, *run(off, adj, w, eps, **opt))


def test_amsf_several_tiles_ragged():
    for off, adj in (gen.rmat(seed=9, scale=15), gen.er(seed=4, n0=70001, pairs=150000, isolated=333),
                     gen.grid(seed=6, rows=301, cols=257)):
        w = gen.exp_weights(off, adj, 2)
        want = oracle.amsf(off, adj, w, 0.25)
        for opt in OPTS[:3]:
            check(off, adj, w, 0.25, *run(off, adj, w, 0.25, **opt), want=want)


def test_amsf_equal_weights_exact_and_ties():
    off, adj = gen.er(seed=5, n0=3000, pairs=5000, isolated=2)
    w = np.full(adj.size, 0.75, dtype=np.float32)
    E, W, tot = run(off, adj, w, 0.25)
    check(off, adj, w, 0.25, E, W, tot)
    assert tot == pytest.approx(oracle.kruskal(off, adj, w)[0], rel=1e-12)      # one bucket: exact
    # integer weights 1..4 with eps = 1: buckets [1,2) [2,4) [4,8): many ties
    w = (1 + (np.arange(adj.size) % 4)).astype(np.float32)
    src = np.repeat(np.arange(off.size - 1), np.diff(off))
    w = (1 + ((np.minimum(src, adj) * 7 + np.maximum(src, adj)) % 4)).astype(np.float32)   # symmetric
    check(off, adj, w, 1.0, *run(off, adj, w, 1.0))


def test_amsf_rejects_bad_input():
    off, adj = gen.er(seed=6, n0=100, pairs=300, isolated=0)
    d_off, d_adj = to_dev(off, adj)
    for bad in (0.0, -1.0, np.inf, np.nan):
        w = gen.exp_weights(off, adj, 1)
        w[5] = bad
        with pytest.raises(cc.CCError):
            pkg.amsf(d_off, d_adj, torch.from_numpy(w).cuda(), 0.25)
    w = torch.from_numpy(gen.exp_weights(off, adj, 1)).cuda()
    for eps in (0.0, -0.5, float("inf")):
        with pytest.raises(cc.CCError):
            pkg.amsf(d_off, d_adj, w, eps)


def test_amsf_counters():
    off, adj = gen.rmat(seed=10, scale=13)
    w = gen.exp_weights(off, adj, 10)
    d_off, d_adj = to_dev(off, adj)
    d_w = torch.from_numpy(w).cuda()
    ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
    E, W, tot = pkg.amsf(d_off, d_adj, d_w, 0.25, counters=ctr)
    c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
    want = oracle.amsf(off, adj, w, 0.25)
    assert c["amsf_rounds"] == want["nbuckets"]
    assert c["amsf_hooks"] == E.shape[0] == want["pairs"].shape[0]
    ctr.zero_()
    pkg.amsf(d_off, d_adj, d_w, 0.25, counters=ctr, flags=cc.FLAG_AMSF_PLAIN | cc.FLAG_NO_SKIP)
    c2 = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
    # plain NF without the skip inspects every adjacency entry in every round
    assert c2["amsf_edges"] == adj.size * want["nbuckets"]
    assert c["amsf_edges"] < c2["amsf_edges"]


def test_amsf_repeat_stress():
    off, adj = gen.rmat(seed=11, scale=12)
    w = gen.exp_weights(off, adj, 11)
    want = oracle.amsf(off, adj, w, 0.25)
    rng = np.random.default_rng(3)
    for it in range(40):
        opt = OPTS[int(rng.integers(0, len(OPTS)))]
        check(off, adj, w, 0.25, *run(off, adj, w, 0.25, **opt), want=want, exact_opt=(it % 10 == 0))


def test_amsf_unaligned_weights():
    """A weight buffer that is not 16-byte aligned takes the scalar sweep."""
    off, adj = gen.rmat(seed=12, scale=13)
    w = gen.exp_weights(off, adj, 12)
    d_off, d_adj = to_dev(off, adj)
    buf = torch.empty(adj.size + 1, dtype=torch.float32, device="cuda")
    buf[1:] = torch.from_numpy(w).cuda()
    E, W, tot = pkg.amsf(d_off, d_adj, buf[1:], 0.25)
    check(off, adj, w, 0.25, u32(E).reshape(-1, 2), W.cpu().numpy(), tot)


def test_amsf_hubs_bucket_index():
    """Lists far longer than the 2048-entry piece size (hub bucket index, several
    pieces per bucket), with and without the index, with and without the skip."""
    rng = np.random.default_rng(5)
    n = 30000
    pairs = [(0, v) for v in range(1, 12001)] + [(1, v) for v in range(2, 30000, 3)]
    pairs += [tuple(rng.integers(0, n, 2)) for _ in range(20000)]
    off, adj = oracle.csr_from_pairs(n, pairs)
    assert np.diff(off).max() > 4 * 2048
    for seed, eps in ((1, 0.25), (2, 0.05), (3, 1.0)):
        w = gen.exp_weights(off, adj, seed)
        want = oracle.amsf(off, adj, w, eps)
        for opt in (OPTS[0], OPTS[1], OPTS[6], dict(flags=cc.FLAG_HALVE)):
            check(off, adj, w, eps, *run(off, adj, w, eps, **opt), want=want)


def test_amsf_chain_shaped():
    """A path whose weights grow along it: every bucket hooks the next stretch under
    the previous one (one long chain); the finds must stay exact and fast."""
    import time
    n = 1 << 18
    ids = np.arange(n - 1, dtype=np.uint64)
    off, adj = oracle.csr_from_pairs(n, np.stack([ids, ids + 1], 1))
    src = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off))
    w = (1.0 + np.minimum(src, adj.astype(np.uint64)).astype(np.float64) / 1000.0).astype(np.float32)
    want = oracle.amsf(off, adj, w, 0.25)
    for opt in (OPTS[0], OPTS[1]):
        t0 = time.time()
        E, W, tot = run(off, adj, w, 0.25, **opt)
        assert time.time() - t0 < 10.0
        check(off, adj, w, 0.25, E, W, tot, want=want)


def test_amsf_host_buffers():
    """Pageable numpy arrays and pinned tensors are staged; results equal the device call."""
    off, adj = gen.rmat(seed=13, scale=12)
    w = gen.exp_weights(off, adj, 13)
    n, m = off.size - 1, adj.size
    d_off, d_adj = to_dev(off, adj)
    E0, W0, t0 = pkg.amsf(d_off, d_adj, torch.from_numpy(w).cuda(), 0.25)
    want = (u32(E0).reshape(-1, 2), W0.cpu().numpy(), t0)
    # pageable host (numpy) everywhere
    edges = np.zeros((n, 2), dtype=np.uint32)
    ew = np.zeros(n, dtype=np.float32)
    num = np.zeros(1, dtype=np.int64)
    tot = np.zeros(1, dtype=np.float64)
    cc.cc_amsf(off, adj, w, n, m, 0.25, edges, ew, num, tot)
    k = int(num[0])
    check(off, adj, w, 0.25, edges[:k], ew[:k], float(tot[0]))
    assert k == want[0].shape[0]
    # pinned host inputs, device outputs
    p_off = torch.from_numpy(off).pin_memory()
    p_adj = torch.from_numpy(adj.view(np.int32)).pin_memory()
    p_w = torch.from_numpy(w).pin_memory()
    d_e = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    d_num = torch.zeros(1, dtype=torch.int64, device="cuda")
    cc.cc_amsf(p_off, p_adj, p_w, n, m, 0.25, d_e, None, d_num, None)
    torch.cuda.synchronize()
    assert int(d_num.item()) == k


def test_amsf_self_loops_extreme_weights():
    """Self-loops carrying the smallest and the largest weight: they set W_min / W_max and
    so the bucket boundaries on both sides (reading R25) but never join the forest."""
    rng = np.random.default_rng(21)
    off, adj = gen.er(seed=11, n0=20000, pairs=30000, isolated=5)
    n = off.size - 1
    loops = rng.choice(n, 300, replace=False)
    pairs = np.concatenate([np.stack([np.repeat(np.arange(n), np.diff(off)), adj.astype(np.int64)], 1),
                            np.stack([loops, loops], 1)])
    off, adj = oracle.csr_from_pairs(n, pairs)
    w = gen.exp_weights(off, adj, 5)
    src = np.repeat(np.arange(n), np.diff(off))
    is_loop = np.nonzero(src == adj)[0]
    assert is_loop.size >= 300
    w[is_loop[0]] = np.float32(w.min() / 1000)
    w[is_loop[1]] = np.float32(w.max() * 1000)
    for eps in (0.05, 0.25):
        want = oracle.amsf(off, adj, w, eps)
        for opt in OPTS:
            E, W, tot = run(off, adj, w, eps, **opt)
            assert not np.any(E[:, 0] == E[:, 1])
            check(off, adj, w, eps, E, W, tot, want=want)


def test_amsf_bucket_boundaries_exact():
    """Weights placed exactly at the bucket boundaries: for b_i = W_min (1+eps)^i (fp64 chain,
    reading R25) the smallest float >= b_i must land in bucket i and the float just below it in
    bucket i-1 -- through the scanned lists, the warp-built index (lists of 257..4096) and the
    CTA-built index (longer lists), whose float thresholds must decide as b_i <= (double)w."""
    eps = 0.1
    b = oracle.amsf_bounds(1.0, 50.0, eps)
    vals = [np.float32(1.0)]
    for bi in b[1:-1]:
        f = np.float32(bi)
        if float(f) < bi:
            f = np.nextafter(f, np.float32(np.inf))
        vals += [f, np.nextafter(f, np.float32(0))]
    vals = np.array(vals, dtype=np.float32)
    for leaves in (40, 1000, 6000):                      # scanned / warp index / CTA index
        n = leaves + 1 + 2
        rng = np.random.default_rng(leaves)
        pairs = [(0, i) for i in range(1, leaves + 1)] + [(leaves + 1, leaves + 2)]
        off, adj = oracle.csr_from_pairs(n, np.array(pairs))
        wmap = {}
        for u, v in pairs:
            wmap[(u, v)] = wmap[(v, u)] = vals[rng.integers(0, vals.size)]
        wmap[(leaves + 1, leaves + 2)] = wmap[(leaves + 2, leaves + 1)] = np.float32(1.0)   # W_min = 1
        src = np.repeat(np.arange(n), np.diff(off))
        w = np.array([wmap[(int(a), int(c))] for a, c in zip(src, adj)], dtype=np.float32)
        want = oracle.amsf(off, adj, w, eps)
        for opt in (OPTS[0], OPTS[6], OPTS[2]):
            check(off, adj, w, eps, *run(off, adj, w, eps, **opt), want=want)
