"""Pins for the CPU oracle (oracle/) against things other than itself.

Each check is chosen so that a plausible slip in the oracle (a dropped edge
direction, a wrong label choice, an off-by-one in the CSR walk, a transposed
pair, a forest check that misses a cycle) fails at least one of them:

* brute-force reachability (Warshall closure) on EVERY labelled graph with
  n <= 5 vertices and on random graphs up to n = 64;
* closed forms: disjoint cliques, disjoint paths, a star, a full grid, the
  edgeless graph, the paper's counter-example graph (App. A.2.3)
  whose correct answer is one component;
* scipy.sparse.csgraph.connected_components (a library routine) partitions;
* the BFS oracle and the DSU oracle agree (two independent constructions);
* forest_check accepts forced forests (trees, the counter-example edge set)
  and rejects each planted defect;
* incr_run against brute-force reachability after every batch, plus the
  closed forms of P:955-958 / reading R15 and the stream/static equivalence.
"""
import itertools

import numpy as np
import pytest

import oracle
from inputs import gen

# ---------------------------------------------------------------------------
# helpers written independently of the oracle (pure Python / numpy)


def csr(n, pairs):
    adjl = [set() for _ in range(n)]
    for u, v in pairs:
        if u != v:
            adjl[u].add(v)
            adjl[v].add(u)
    off = np.zeros(n + 1, dtype=np.int64)
    for i in range(n):
        off[i + 1] = off[i] + len(adjl[i])
    adj = np.array([x for i in range(n) for x in sorted(adjl[i])], dtype=np.uint32)
    return off, adj


def warshall_labels(n, pairs):
    """lab[v] = min{j : j reachable from v} by transitive closure."""
    R = np.eye(n, dtype=bool)
    for u, v in pairs:
        R[u, v] = R[v, u] = True
    for k in range(n):
        R |= R[:, k:k + 1] & R[k:k + 1, :]
    return np.array([int(np.argmax(R[v])) for v in range(n)], dtype=np.uint32)


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_exhaustive_small_graphs(n):
    all_pairs = list(itertools.combinations(range(n), 2))
    for mask in range(1 << len(all_pairs)):
        pairs = [p for i, p in enumerate(all_pairs) if mask >> i & 1]
        off, adj = csr(n, pairs)
        want = warshall_labels(n, pairs)
        assert np.array_equal(oracle.cc_bfs(off, adj), want), (n, pairs)
        assert np.array_equal(oracle.cc_dsu(off, adj), want), (n, pairs)


def test_random_graphs_vs_warshall():
    rng = np.random.default_rng(12345)
    for trial in range(200):
        n = int(rng.integers(1, 65))
        m = int(rng.integers(0, 2 * n + 1))
        pairs = [tuple(int(x) for x in rng.integers(0, n, 2)) for _ in range(m)]
        off, adj = csr(n, pairs)
        want = warshall_labels(n, pairs)
        assert np.array_equal(oracle.cc_bfs(off, adj), want), trial
        assert np.array_equal(oracle.cc_dsu(off, adj), want), trial


# ---------------------------------------------------------------------------
# closed forms
def test_disjoint_cliques():
    t, s = 7, 5
    pairs = [(b * s + i, b * s + j) for b in range(t) for i in range(s) for j in range(i + 1, s)]
    off, adj = csr(t * s, pairs)
    want = (np.arange(t * s) // s * s).astype(np.uint32)
    assert np.array_equal(oracle.cc_bfs(off, adj), want)
    assert np.array_equal(oracle.cc_dsu(off, adj), want)


def test_disjoint_paths_reversed_ids():
    # paths laid out in decreasing id order inside each block: the minimum is the path's last vertex
    t, s = 4, 9
    pairs = [(b * s + i + 1, b * s + i) for b in range(t) for i in range(s - 1)]
    off, adj = csr(t * s, pairs)
    want = (np.arange(t * s) // s * s).astype(np.uint32)
    assert np.array_equal(oracle.cc_bfs(off, adj), want)


def test_star_center_last():
    n = 50
    pairs = [(n - 1, i) for i in range(n - 1)]
    off, adj = csr(n, pairs)
    assert np.array_equal(oracle.cc_bfs(off, adj), np.zeros(n, dtype=np.uint32))
    assert np.array_equal(oracle.cc_dsu(off, adj), np.zeros(n, dtype=np.uint32))


def test_full_grid_one_component():
    R, C = 17, 23
    pairs = [(r * C + c, r * C + c + 1) for r in range(R) for c in range(C - 1)]
    pairs += [(r * C + c, (r + 1) * C + c) for r in range(R - 1) for c in range(C)]
    off, adj = csr(R * C, pairs)
    assert np.array_equal(oracle.cc_bfs(off, adj), np.zeros(R * C, dtype=np.uint32))
    # grid generator with p = 1 keeps every candidate edge: also one component
    off2, adj2 = gen.grid(seed=9, rows=R, cols=C, p32=1 << 32)
    assert np.array_equal(off2, off) and np.array_equal(adj2, adj)


def test_edgeless_and_isolated_tail():
    off = np.zeros(10, dtype=np.int64)
    adj = np.zeros(0, dtype=np.uint32)
    assert np.array_equal(oracle.cc_bfs(off, adj), np.arange(9, dtype=np.uint32))
    assert np.array_equal(oracle.cc_dsu(off, adj), np.arange(9, dtype=np.uint32))
    # ER with 0 draws plus isolated vertices: identity
    off, adj = gen.er(seed=1, n0=100, pairs=0, isolated=10)
    assert np.array_equal(oracle.cc_bfs(off, adj), np.arange(110, dtype=np.uint32))


COUNTER_EXAMPLE = [(0, 2), (1, 3), (2, 5), (3, 4), (4, 5)]


def test_paper_counter_example_graph():
    """App. A.2.3: the excluded combination answers 2; the truth is 1."""
    off, adj = csr(6, COUNTER_EXAMPLE)
    lab = oracle.cc_bfs(off, adj)
    assert np.array_equal(lab, np.zeros(6, dtype=np.uint32))
    assert len(set(lab.tolist())) == 1
    # a path 0-2-5-4-3-1 is a tree: its spanning forest is E itself (n - c = 5 edges)
    assert oracle.forest_check(off, adj, 1, np.array(COUNTER_EXAMPLE))[0] == 0


# ---------------------------------------------------------------------------
def test_scipy_partition_and_cross_oracle():
    sp = pytest.importorskip("scipy.sparse")
    csgraph = pytest.importorskip("scipy.sparse.csgraph")
    graphs = [gen.er(), gen.grid(seed=2, rows=256, cols=256), gen.rmat(seed=3, scale=14)]
    for off, adj in graphs:
        n = off.size - 1
        lab = oracle.cc_bfs(off, adj)
        assert np.array_equal(lab, oracle.cc_dsu(off, adj))
        A = sp.csr_matrix((np.ones(adj.size, dtype=np.int8), adj.astype(np.int64), off), shape=(n, n))
        nc, sl = csgraph.connected_components(A, directed=False)
        assert nc == int(np.sum(lab == np.arange(n)))
        # same partition: the map scipy-label -> oracle-label is a bijection
        pairs = np.unique(np.stack([sl, lab.astype(np.int64)], 1), axis=0)
        assert pairs.shape[0] == nc
        # canonical form invariants (reading R13)
        assert np.all(lab <= np.arange(n))
        assert np.array_equal(lab[lab], lab)


# ---------------------------------------------------------------------------
def bfs_forest(n, pairs):
    off, adj = csr(n, pairs)
    seen = [False] * n
    F = []
    for s in range(n):
        if seen[s]:
            continue
        seen[s] = True
        q = [s]
        while q:
            x = q.pop()
            for e in range(off[x], off[x + 1]):
                y = int(adj[e])
                if not seen[y]:
                    seen[y] = True
                    F.append((y, x))
                    q.append(y)
    return off, adj, F


def test_forest_check_accepts_valid_and_rejects_defects():
    rng = np.random.default_rng(7)
    n = 40
    pairs = [tuple(int(x) for x in rng.integers(0, n, 2)) for _ in range(60)]
    off, adj, F = bfs_forest(n, pairs)
    c = int(np.sum(warshall_labels(n, pairs) == np.arange(n)))
    assert len(F) == n - c
    assert oracle.forest_check(off, adj, c, np.array(F)) == (0, -1)
    # (1) count
    assert oracle.forest_check(off, adj, c, np.array(F[:-1]))[0] == 1
    # (2) out of range
    bad = list(F)
    bad[3] = (n, bad[3][1])
    assert oracle.forest_check(off, adj, c, np.array(bad)) == (2, 3)
    # (3) self-loop
    bad = list(F)
    bad[5] = (bad[5][0], bad[5][0])
    assert oracle.forest_check(off, adj, c, np.array(bad)) == (3, 5)
    # (4) a non-edge (transposition-safe: check a pair that is not adjacent)
    non_edges = [(u, v) for u in range(n) for v in range(n) if u != v and v not in set(adj[off[u]:off[u + 1]].tolist())]
    bad = list(F)
    bad[0] = non_edges[0]
    assert oracle.forest_check(off, adj, c, np.array(bad))[0] in (4,)
    # (5) a cycle: replace the last forest edge with a graph edge closing a cycle
    Fs = set(F) | {(b, a) for a, b in F}
    extra = [(u, int(v)) for u in range(n) for v in adj[off[u]:off[u + 1]] if (u, int(v)) not in Fs]
    assert extra, "fixture must have a non-tree edge"
    bad = list(F[:-1]) + [extra[0]]
    rc, idx = oracle.forest_check(off, adj, c, np.array(bad))
    # dropping one tree edge and adding a non-tree edge either closes a cycle, or
    # (if the non-tree edge reconnects the split) forms another valid forest
    assert rc in (0, 5)
    # a guaranteed cycle: forest + the extra edge, minus nothing, with the count fudged
    rc, idx = oracle.forest_check(off, adj, c - 1, np.array(F + [extra[0]]))
    assert rc == 5 and idx == len(F)


def test_forest_check_tree_forced():
    # a tree on 10 vertices: its only spanning forest is its edge set (SPEC S:385-392 example)
    pairs = [(i, (i - 1) // 2) for i in range(1, 10)]
    off, adj = csr(10, pairs)
    assert oracle.forest_check(off, adj, 1, np.array(pairs))[0] == 0
    assert oracle.forest_check(off, adj, 1, np.array([(b, a) for a, b in pairs]))[0] == 0
    # edgeless: empty forest, n components
    off0 = np.zeros(6, dtype=np.int64)
    assert oracle.forest_check(off0, np.zeros(0, np.uint32), 5, np.zeros((0, 2), np.uint32))[0] == 0


# ---------------------------------------------------------------------------
def test_incr_vs_bruteforce_each_batch():
    rng = np.random.default_rng(3)
    for trial in range(30):
        n = int(rng.integers(1, 30))
        nb = int(rng.integers(1, 6))
        batches, all_ins = [], []
        for _ in range(nb):
            ins = rng.integers(0, n, (int(rng.integers(0, 8)), 2))
            qs = rng.integers(0, n, (int(rng.integers(0, 8)), 2))
            batches.append((ins, qs))
        ans, lab = oracle.incr_run(n, batches, want_labels=True)
        pos = 0
        for ins, qs in batches:
            all_ins += [tuple(int(x) for x in p) for p in ins]
            w = warshall_labels(n, all_ins)          # reading R15: own batch's inserts visible
            for a, b in qs:
                assert ans[pos] == (1 if w[a] == w[b] else 0)
                pos += 1
        assert pos == ans.size
        assert np.array_equal(lab, warshall_labels(n, all_ins))


def test_incr_closed_forms_and_monotone():
    n = 16
    batches = [
        (np.array([[0, 1], [1, 2]]), np.array([[0, 2], [3, 3], [0, 3]])),   # SPEC S:466 example
        (np.array([[2, 3]]), np.array([[0, 3], [5, 9], [3, 0]])),
        (np.zeros((0, 2), int), np.array([[0, 2], [0, 3], [7, 7]])),
    ]
    ans, _ = oracle.incr_run(n, batches)
    assert ans.tolist() == [1, 1, 0, 1, 0, 1, 1, 1, 1]


def test_incr_final_labels_equal_static():
    off, adj = gen.rmat(seed=5, scale=10)
    n = off.size - 1
    src = np.repeat(np.arange(n), np.diff(off))
    pairs = np.stack([src, adj.astype(np.int64)], 1)
    pairs = pairs[pairs[:, 0] < pairs[:, 1]]
    rng = np.random.default_rng(0)
    rng.shuffle(pairs)
    for bs in (1, 10, 1000, pairs.shape[0]):
        batches = [(pairs[i:i + bs], np.zeros((0, 2), int)) for i in range(0, pairs.shape[0], bs)]
        _, lab = oracle.incr_run(n, batches, want_labels=True)
        assert np.array_equal(lab, oracle.cc_bfs(off, adj))


# ---------------------------------------------------------------------------
def test_kout_sample_edges_closed_forms():
    # star ordered by id: every vertex's first neighbour is 0 -> one component
    n = 30
    off, adj = csr(n, [(0, i) for i in range(1, n)] + [(i, i + 1) for i in range(1, n - 1)])
    E = oracle.kout_sample_edges(off, adj, 1, "afforest")
    assert E.shape == (n, 2) and np.all(E[1:, 1] == 0)
    o2, a2 = oracle.csr_from_pairs(n, E)
    assert np.array_equal(oracle.cc_bfs(o2, a2), np.zeros(n, dtype=np.uint32))
    # afforest: sum_u min(k, deg u) edges; positions are the first k of each list
    off, adj = gen.rmat(seed=11, scale=12)
    deg = np.diff(off)
    for k in (1, 2, 3):
        E = oracle.kout_sample_edges(off, adj, k, "afforest")
        assert E.shape[0] == int(np.minimum(deg, k).sum())
    # hybrid: first edge + k-1 picks inside each list; identical to afforest when deg <= 1
    E = oracle.kout_sample_edges(off, adj, 2, "hybrid", seed=5)
    assert E.shape[0] == 2 * int((deg > 0).sum())
    for u, v in E[:2000]:
        assert v in set(adj[off[u]:off[u + 1]].tolist())
    # hybrid's first pick is the first neighbour; pure draws every pick
    first = set(zip(np.nonzero(deg > 0)[0].tolist(), adj[off[:-1][deg > 0]].tolist()))
    assert first <= set(map(tuple, E.tolist()))
    Ep = oracle.kout_sample_edges(off, adj, 3, "pure", seed=5)
    assert Ep.shape[0] == 3 * int((deg > 0).sum())
    for u, v in Ep[::97]:
        assert v in set(adj[off[u]:off[u + 1]].tolist())
    # a vertex of degree 1 samples its only edge under every variant
    d1 = np.nonzero(deg == 1)[0][:50]
    for var in ("afforest", "hybrid", "pure"):
        Ev = oracle.kout_sample_edges(off, adj, 2, var, seed=1)
        got = set(map(tuple, Ev.tolist()))
        assert all((int(u), int(adj[off[u]])) in got for u in d1)


def test_identify_frequent_and_canon():
    assert oracle.identify_frequent(np.full(100, 7, dtype=np.uint32), 1024, 1) == 7
    lab = np.zeros(1000, dtype=np.uint32)
    lab[900:] = 900
    assert oracle.identify_frequent(lab, 1024, 3) == 0
    assert np.array_equal(oracle.canon([2, 2, 2]), [0, 0, 0])
    assert np.array_equal(oracle.canon([5, 5, 1, 1, 4]), [0, 0, 2, 2, 4])
    assert np.array_equal(oracle.canon(np.arange(9)), np.arange(9))
    # splitmix64 published test vector (seed 0 -> first output), pins the shared generator form
    assert int(oracle.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_kout_sample_edges_pins():
    """Pins of the k-out sample beyond its own definition (R7): afforest with k >= max degree
    samples every edge (its CC is scipy's); hybrid/pure picks are uniform over the list
    positions and independent across j (chi-square, "uniformly at random")."""
    from scipy import stats
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components
    off, adj = gen.er(seed=13, n0=3000, pairs=4000, isolated=7)
    n = off.size - 1
    deg = np.diff(off)
    E = oracle.kout_sample_edges(off, adj, int(deg.max()), "afforest")
    src = np.repeat(np.arange(n), deg)
    assert set(zip(E[:, 0].tolist(), E[:, 1].tolist())) == set(zip(src.tolist(), adj.tolist()))
    g = csr_matrix((np.ones(E.shape[0]), (E[:, 0], E[:, 1])), shape=(n, n))
    nc, lab = connected_components(g, directed=False)
    assert nc == int(np.sum(oracle.cc_bfs(off, adj) == np.arange(n)))
    # circulant graph: every list is the same 12 offsets, so the position of a pick is its rank
    n, d = 20000, 12
    ring = [(u, (u + s) % n) for u in range(n) for s in range(1, d // 2 + 1)]
    off, adj = oracle.csr_from_pairs(n, np.array(ring))
    assert np.all(np.diff(off) == d)
    for var, k in (("hybrid", 3), ("pure", 2)):
        E = oracle.kout_sample_edges(off, adj, k, var, seed=7)
        assert E.shape[0] == k * n
        u = E[:, 0].astype(np.int64)
        pos = np.array([np.searchsorted(adj[off[a]:off[a + 1]], b) for a, b in zip(u, E[:, 1])])
        # picks are in u's list (searchsorted found them) and grouped by j in blocks of n
        assert np.all(adj[off[u] + pos] == E[:, 1])
        first = 1 if var == "hybrid" else 0
        if var == "hybrid":
            assert np.all(pos[:n] == 0)
        picks = pos[first * n:].reshape(k - first, n)
        for j in range(picks.shape[0]):
            assert stats.chisquare(np.bincount(picks[j], minlength=d)).pvalue > 1e-4
        if picks.shape[0] >= 2:
            pairs = picks[0] * d + picks[1]
            assert stats.chisquare(np.bincount(pairs, minlength=d * d)).pvalue > 1e-4


def test_uniform_below_and_identify_frequent_pins():
    """uniform_below is the multiply-shift map: value x has preimage [ceil(x 2^32 / b),
    ceil((x+1) 2^32 / b)) of the low 32 bits (sizes differ by <= 1); IdentifyFrequent is the
    mode of the sampled labels with ties to the smaller label (R9), i.e. scipy.stats.mode."""
    from scipy import stats
    for b in (1, 2, 3, 7, 1000, 4096, 134217728, 0xFFFFFFFF):
        for x in {x for x in (0, 1, b // 2, b - 1) if x < b}:
            lo = -(-(x * (1 << 32)) // b)                         # ceil(x 2^32 / b)
            assert int(oracle.uniform_below(np.array([lo], dtype=np.uint64), b)[0]) == x
            if lo > 0:
                assert int(oracle.uniform_below(np.array([lo - 1], dtype=np.uint64), b)[0]) == x - 1
        hi = np.array([(1 << 64) - 1], dtype=np.uint64)           # high bits are ignored
        assert int(oracle.uniform_below(hi, b)[0]) == b - 1
    # sample positions: in range, uniform (chi-square), distinct seeds give distinct draws
    pos = oracle.sample_positions(1000, 200000, 3)
    assert pos.min() >= 0 and pos.max() < 1000
    assert stats.chisquare(np.bincount(pos, minlength=1000)).pvalue > 1e-4
    assert not np.array_equal(oracle.sample_positions(1000, 1024, 3), oracle.sample_positions(1000, 1024, 4))
    rng = np.random.default_rng(5)
    for t in range(200):
        n = int(rng.integers(1, 300))
        lab = rng.integers(0, int(rng.integers(1, 6)), n).astype(np.uint32)   # few labels: many ties
        s = int(rng.integers(1, 64))
        vals = lab[oracle.sample_positions(n, s, t)]
        assert oracle.identify_frequent(lab, s, t) == int(stats.mode(vals, keepdims=False).mode)
    # a 60 % giant is the mode of 1024 samples for every seed (a 40 % rival would need > 512 hits)
    lab = np.where(np.arange(100000) % 5 < 3, 3, 8).astype(np.uint32)
    assert all(oracle.identify_frequent(lab, 1024, s) == 3 for s in range(50))


def test_golden_fixtures():
    """tests/golden/: the paper's worked graph (App. A.2.3) and a forest-size fixture, each
    with the values the paper fixes for it (one component; n - c forest edges)."""
    from tests.helpers import golden_fixtures
    seen = 0
    for name, off, adj, want in golden_fixtures():
        n = off.size - 1
        lab = oracle.cc_bfs(off, adj)
        assert np.array_equal(lab, want["labels"]), name
        assert int(np.sum(lab == np.arange(n))) == want["components"], name
        assert np.array_equal(oracle.cc_dsu(off, adj), want["labels"]), name
        assert n - want["components"] == want["forest_edges"], name
        seen += 1
    assert seen >= 2
