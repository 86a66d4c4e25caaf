"""GPU parity of the static path (cc_labels, cc_spanning_forest) vs the CPU oracle.

Bit-exact: labels are compared raw (canonical min-id form, reading R13) to
oracle.cc_bfs.  Forests: the oracle's validity triple plus bit-exact labels.
All calls go through the C ABI (libcc.so via paper_2008_03909_b200.cc).
"""
import itertools

import numpy as np
import pytest

import oracle
from inputs import gen
from tests.helpers import csr, fixtures, to_dev, u32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2008_03909_b200 as pkg  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402

OPTION_GRID = [
    dict(k=2, variant="afforest", flags=0),
    dict(k=0, variant="afforest", flags=0),
    dict(k=1, variant="afforest", flags=0),
    dict(k=3, variant="afforest", flags=0),
    dict(k=2, variant="hybrid", flags=0, seed=7),
    dict(k=3, variant="hybrid", flags=0, seed=11),
    dict(k=2, variant="afforest", flags=cc.FLAG_HALVE),
    dict(k=2, variant="afforest", flags=cc.FLAG_UF_ASYNC),
    dict(k=2, variant="afforest", flags=cc.FLAG_NO_SKIP),
    dict(k=2, variant="afforest", flags=cc.FLAG_NO_DEGSKIP | cc.FLAG_NO_MIDCOMPRESS),
    dict(k=64, variant="afforest", flags=0),
    dict(k=2, variant="afforest", flags=cc.FLAG_MIDCOMPRESS),
    dict(k=3, variant="hybrid", flags=cc.FLAG_MIDCOMPRESS | cc.FLAG_HALVE, seed=5),
    dict(k=2, variant="pure", flags=0, seed=13),
    dict(k=2, variant="afforest", flags=cc.FLAG_FINISH_SV),
    dict(k=0, variant="afforest", flags=cc.FLAG_FINISH_SV),
    dict(k=1, variant="hybrid", flags=cc.FLAG_FINISH_SV | cc.FLAG_NO_SKIP, seed=3),
    dict(k=1, variant="pure", flags=cc.FLAG_UF_ASYNC, seed=2),
    # the contracted k-out link and the round-1 (no lane refill) link kernel
    dict(k=2, variant="afforest", flags=cc.FLAG_CONTRACT),
    dict(k=3, variant="hybrid", flags=cc.FLAG_CONTRACT | cc.FLAG_HALVE, seed=5),
    dict(k=2, variant="pure", flags=cc.FLAG_CONTRACT | cc.FLAG_UF_ASYNC, seed=9),
    dict(k=2, variant="afforest", flags=cc.FLAG_NO_REFILL),
    dict(k=3, variant="hybrid", flags=cc.FLAG_NO_REFILL, seed=3),
    # sampling and k-out links in one kernel
    dict(k=2, variant="afforest", flags=cc.FLAG_FUSED_LINK),
    dict(k=1, variant="afforest", flags=cc.FLAG_FUSED_LINK),
    dict(k=2, variant="hybrid", flags=cc.FLAG_FUSED_LINK, seed=4),
    dict(k=2, variant="pure", flags=cc.FLAG_FUSED_LINK | cc.FLAG_NO_DEGSKIP, seed=8),
    # Liu-Tarjan CRFA finish (NEXT-3)
    dict(k=2, variant="afforest", flags=cc.FLAG_FINISH_CRFA),
    dict(k=0, variant="afforest", flags=cc.FLAG_FINISH_CRFA),
    dict(k=1, variant="hybrid", flags=cc.FLAG_FINISH_CRFA | cc.FLAG_NO_SKIP, seed=3),
]


def run_labels(off, adj, **kw):
    d_off, d_adj = to_dev(off, adj)
    lab = pkg.connected_components(d_off, d_adj, **kw)
    torch.cuda.synchronize()
    return u32(lab)


def small_graphs():
    G = [(name, off, adj) for name, off, adj in fixtures()]
    G.append(("er_small", *gen.er(seed=3, n0=5000, pairs=6000, isolated=37)))
    G.append(("er_sparse", *gen.er(seed=4, n0=20000, pairs=9000, isolated=5)))
    G.append(("grid_ragged", *gen.grid(seed=5, rows=67, cols=131)))
    G.append(("rmat10", *gen.rmat(seed=6, scale=10)))
    G.append(("rmat13_unperm", *gen.rmat(seed=7, scale=13, permuted=False)))
    return G


@pytest.mark.parametrize("opt", OPTION_GRID, ids=lambda o: f"k{o['k']}-{o['variant']}-f{o['flags']}")
def test_labels_bit_exact_small(opt):
    for name, off, adj in small_graphs():
        want = oracle.cc_bfs(off, adj)
        got = run_labels(off, adj, **opt)
        assert np.array_equal(got, want), (name, opt, np.nonzero(got != want)[0][:5])


@pytest.mark.parametrize("scale", [12, 15])
def test_labels_rmat_several_tiles(scale):
    off, adj = gen.rmat(seed=8, scale=scale)
    want = oracle.cc_bfs(off, adj)
    for opt in OPTION_GRID[:6]:
        assert np.array_equal(run_labels(off, adj, **opt), want), opt


def test_labels_grid_and_er_mid():
    for off, adj in (gen.grid(seed=2, rows=512, cols=384), gen.er(seed=1)):
        want = oracle.cc_bfs(off, adj)
        for opt in (OPTION_GRID[0], OPTION_GRID[1], OPTION_GRID[4]):
            assert np.array_equal(run_labels(off, adj, **opt), want), opt


# ---------------------------------------------------------------------------
def test_sampled_labels_are_cc_of_the_sampled_edges():
    """H2+H3: after the sampling compress, P is height-one (Def. 3.1)
    and -- by the min-root invariant -- equals the canonical CC labels of the
    sampled edge set (Alg. 4); H4 returns the mode of the seeded samples."""
    graphs = [gen.rmat(seed=9, scale=12), gen.grid(seed=3, rows=100, cols=77), gen.er(seed=2, n0=3000, pairs=4000)]
    graphs += [(o, a) for _, o, a in fixtures()]
    for off, adj in graphs:
        n = off.size - 1
        for (k, variant, seed), fl in itertools.product(
                [(1, "afforest", 0), (2, "afforest", 0), (3, "afforest", 0), (2, "hybrid", 5),
                 (4, "hybrid", 99), (1, "pure", 4), (3, "pure", 8)],
                [0, cc.FLAG_CONTRACT, cc.FLAG_NO_REFILL, cc.FLAG_FUSED_LINK]):
            d_off, d_adj = to_dev(off, adj)
            sampled = torch.empty(n, dtype=torch.int32, device="cuda")
            lmax = torch.empty(1, dtype=torch.int32, device="cuda")
            lab = pkg.connected_components(d_off, d_adj, k=k, variant=variant, seed=seed, sampled_out=sampled,
                                           lmax_out=lmax, flags=fl)
            E = oracle.kout_sample_edges(off, adj, k, variant, seed)
            o2, a2 = oracle.csr_from_pairs(n, E)
            want_s = oracle.cc_bfs(o2, a2)
            got_s = u32(sampled)
            assert np.array_equal(got_s, want_s), (k, variant)
            assert np.array_equal(got_s[got_s], got_s)                   # height-one
            assert int(u32(lmax)[0]) == oracle.identify_frequent(want_s, 1024, seed)
            assert np.array_equal(u32(lab), oracle.cc_bfs(off, adj))


def test_lmax_forcing_changes_nothing():
    off, adj = gen.rmat(seed=10, scale=12)
    n = off.size - 1
    want = oracle.cc_bfs(off, adj)
    roots = np.unique(want)
    for forced in [int(roots[0]), int(roots[-1]), int(roots[len(roots) // 2]), 0xFFFFFFFF, n - 1, 12345 % n]:
        f = torch.tensor([np.uint32(forced).view(np.int32)], dtype=torch.int32, device="cuda")
        for k in (0, 1, 2):
            d_off, d_adj = to_dev(off, adj)
            lab = pkg.connected_components(d_off, d_adj, k=k, lmax_force=f)
            assert np.array_equal(u32(lab), want), (forced, k)


def test_lmax_forcing_non_roots_every_finish():
    """A forced L_max that is not a root of the sampled forest (cc_opts.lmax_force) must change
    nothing either, for every finish: UF-Rem-CAS, SV and CRFA (whose rounds need a height-one
    P after the scan -- the fuzz campaign found a grid where a non-root L_max broke that),
    with and without the degree skip and with the contracted link."""
    graphs = [gen.grid(seed=3, rows=69, cols=173), gen.grid(seed=4, rows=40, cols=90, p32=3 << 30),
              gen.rmat(seed=10, scale=11)]
    for off, adj in graphs:
        n = off.size - 1
        want = oracle.cc_bfs(off, adj)
        d_off, d_adj = to_dev(off, adj)
        for k in (1, 2):
            sampled = torch.empty(n, dtype=torch.int32, device="cuda")
            pkg.connected_components(d_off, d_adj, k=k, sampled_out=sampled)
            s_lab = u32(sampled)
            nonroots = np.nonzero(s_lab != np.arange(n))[0]
            picks = [int(x) for x in nonroots[:: max(1, nonroots.size // 5)][:5]]
            for forced in picks:
                f = torch.tensor([np.uint32(forced).view(np.int32)], dtype=torch.int32, device="cuda")
                for fl in (0, cc.FLAG_FINISH_SV, cc.FLAG_FINISH_CRFA, cc.FLAG_FINISH_SV | cc.FLAG_NO_DEGSKIP,
                           cc.FLAG_CONTRACT, cc.FLAG_NO_DEGSKIP):
                    lab = pkg.connected_components(d_off, d_adj, k=k, lmax_force=f, flags=fl)
                    assert np.array_equal(u32(lab), want), (n, k, forced, fl)
                    edges, lab2 = pkg.spanning_forest(d_off, d_adj, k=k, lmax_force=f, flags=fl)
                    c = int(np.sum(want == np.arange(n)))
                    assert oracle.forest_check(off, adj, c, u32(edges).reshape(-1, 2))[0] == 0, (k, forced, fl)


def test_permutation_and_list_order_metamorphic():
    off, adj = gen.rmat(seed=12, scale=11, permuted=False)
    n = off.size - 1
    base = oracle.cc_bfs(off, adj)
    rng = np.random.default_rng(0)
    pi = rng.permutation(n).astype(np.uint32)
    src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(off))
    o2, a2 = gen.csr_from_directed_pairs(n, pi[src], pi[adj])
    got = run_labels(o2, a2)
    # canonical labels of the permuted graph = canon(pi(base labels))
    want = oracle.canon(base[np.argsort(pi)])
    assert np.array_equal(got, want)
    # shuffle every adjacency list (first-k edges change; labels must not)
    a3 = adj.copy()
    for v in range(n):
        seg = a3[off[v]:off[v + 1]]
        rng.shuffle(seg)
    for k in (1, 2, 3):
        assert np.array_equal(run_labels(off, a3, k=k), base)


def test_host_buffers_equal_device():
    off, adj = gen.rmat(seed=13, scale=11)
    n = off.size - 1
    out = np.zeros(n, dtype=np.uint32)
    cc.cc_labels(off, adj, n, adj.size, out, cc.make_opts())
    assert np.array_equal(out, oracle.cc_bfs(off, adj))
    edges = np.zeros(2 * n, dtype=np.uint32)
    ne = np.zeros(1, dtype=np.int64)
    lab = np.zeros(n, dtype=np.uint32)
    cc.cc_spanning_forest(off, adj, n, adj.size, edges, ne, lab, cc.make_opts())
    c = int(np.sum(lab == np.arange(n)))
    assert np.array_equal(lab, oracle.cc_bfs(off, adj))
    assert oracle.forest_check(off, adj, c, edges[:2 * ne[0]])[0] == 0


def test_validate_flag_rejects_malformed():
    off, adj = gen.rmat(seed=14, scale=8)
    n = off.size - 1
    bad = adj.copy()
    bad[3] = n + 5
    d_off, d_adj = to_dev(off, bad)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    with pytest.raises(cc.CCError):
        cc.cc_labels(d_off, d_adj, n, bad.size, lab, cc.make_opts(flags=cc.FLAG_VALIDATE))
    off2 = off.copy()
    off2[n // 2] = off2[n // 2 + 1] + 1
    d_off, d_adj = to_dev(off2, adj)
    with pytest.raises(cc.CCError):
        cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(flags=cc.FLAG_VALIDATE))
    d_off, d_adj = to_dev(off, adj)
    cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(flags=cc.FLAG_VALIDATE))
    assert np.array_equal(u32(lab), oracle.cc_bfs(off, adj))


def test_empty_and_degenerate_abi():
    # n = 0: OK, no work
    z = torch.zeros(1, dtype=torch.int64, device="cuda")
    cc.cc_labels(z, None, 0, 0, None)
    num = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    cc.cc_spanning_forest(z, None, 0, 0, None, num)
    assert int(num.item()) == 0
    # m = 0: identity
    off = np.zeros(1001, dtype=np.int64)
    got = run_labels(off, np.zeros(0, dtype=np.uint32))
    assert np.array_equal(got, np.arange(1000, dtype=np.uint32))


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("opt", [OPTION_GRID[0], OPTION_GRID[1], OPTION_GRID[4], OPTION_GRID[6], OPTION_GRID[7],
                                 dict(k=2, variant="afforest", flags=cc.FLAG_FINISH_SV),
                                 dict(k=0, variant="afforest", flags=cc.FLAG_FINISH_SV),
                                 dict(k=2, variant="afforest", flags=cc.FLAG_CONTRACT),
                                 dict(k=3, variant="pure", flags=cc.FLAG_CONTRACT | cc.FLAG_HALVE, seed=4),
                                 dict(k=2, variant="afforest", flags=cc.FLAG_NO_REFILL),
                                 dict(k=2, variant="afforest", flags=cc.FLAG_FUSED_LINK),
                                 dict(k=2, variant="hybrid", flags=cc.FLAG_FUSED_LINK, seed=3),
                                 dict(k=2, variant="afforest", flags=cc.FLAG_FINISH_CRFA),
                                 dict(k=0, variant="afforest", flags=cc.FLAG_FINISH_CRFA),
                                 dict(k=1, variant="hybrid", flags=0, seed=6)],
                         ids=lambda o: f"k{o['k']}-{o['variant']}-f{o['flags']}")
def test_spanning_forest_valid(opt):
    for name, off, adj in small_graphs():
        n = off.size - 1
        want = oracle.cc_bfs(off, adj)
        c = int(np.sum(want == np.arange(n)))
        d_off, d_adj = to_dev(off, adj)
        edges, lab = pkg.spanning_forest(d_off, d_adj, **opt)
        E = u32(edges).reshape(-1, 2)
        rc, bad = oracle.forest_check(off, adj, c, E)
        assert rc == 0, (name, opt, oracle.FOREST_ERRORS[rc], bad)
        assert np.array_equal(u32(lab), want), name
        # each slot holds the edge that hooked root r: emitted in ascending slot order,
        # and the hooked slot (the larger root) is never a final root
        assert E.shape[0] == n - c


def test_spanning_forest_without_labels():
    off, adj = gen.grid(seed=6, rows=90, cols=70)
    n = off.size - 1
    d_off, d_adj = to_dev(off, adj)
    edges, lab = pkg.spanning_forest(d_off, d_adj, with_labels=False)
    assert lab is None
    want = oracle.cc_bfs(off, adj)
    c = int(np.sum(want == np.arange(n)))
    assert oracle.forest_check(off, adj, c, u32(edges))[0] == 0


def test_repeat_stress_random_options():
    """Races must never change the answer: 1,000 repeats (SURVEY 8(c) test matrix)
    with random k, variant, seed, flags AND random launch configurations (every
    grid-strided kernel launched with a random block count, 1 .. 4x the default),
    on fixtures, an ER graph spanning many tiles and C1 (BASELINE configs[0])."""
    import inputs
    graphs = [("er", *gen.er(seed=21, n0=30000, pairs=45000, isolated=11)), ("C1", *gen.er(seed=inputs.C1.seed))]
    graphs += [(nm, o, a) for nm, o, a in fixtures() if nm in ("lmax_merges_smaller", "two_giants", "hubs",
                                                                 "path_decreasing", "dups_and_loops")]
    dev = [(nm, *to_dev(o, a), oracle.cc_bfs(o, a), o, a) for nm, o, a in graphs]
    rng = np.random.default_rng(1)
    flags_pool = [0, cc.FLAG_HALVE, cc.FLAG_UF_ASYNC, cc.FLAG_NO_SKIP, cc.FLAG_NO_MIDCOMPRESS, cc.FLAG_NO_DEGSKIP,
                  cc.FLAG_MIDCOMPRESS, cc.FLAG_FINISH_SV, cc.FLAG_CONTRACT, cc.FLAG_NO_REFILL,
                  cc.FLAG_FINISH_CRFA, cc.FLAG_FUSED_LINK]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    try:
        for it in range(1000):
            name, d_off, d_adj, want, off, adj = dev[it % len(dev)]
            k = int(rng.integers(0, 5))
            variant = ["afforest", "hybrid", "pure"][int(rng.integers(0, 3))]
            fl = int(rng.choice(flags_pool)) | int(rng.choice(flags_pool))
            grid = 0 if it % 7 == 0 else int(rng.integers(1, 4 * 8 * sms + 1))
            cc.set_grid(grid)
            seed = int(rng.integers(0, 1 << 30))
            if it % 5 == 4:
                edges, lab = pkg.spanning_forest(d_off, d_adj, k=k, variant=variant, seed=seed, flags=fl)
                c = int(np.sum(want == np.arange(want.size)))
                rc, bad = oracle.forest_check(off, adj, c, u32(edges).reshape(-1, 2))
                assert rc == 0, (it, name, k, variant, fl, grid, oracle.FOREST_ERRORS[rc])
            else:
                lab = pkg.connected_components(d_off, d_adj, k=k, variant=variant, seed=seed, flags=fl)
            assert np.array_equal(u32(lab), want), (it, name, k, variant, fl, grid)
    finally:
        cc.set_grid(0)


def test_counters_and_timings():
    off, adj = gen.rmat(seed=15, scale=12)
    n = off.size - 1
    d_off, d_adj = to_dev(off, adj)
    ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
    t = cc.Timings()
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(counters=ctr, timings=t))
    c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
    deg = np.diff(off)
    assert c["pending_links"] == int(np.minimum(deg, 2).sum()) - int(
        sum(1 for v in range(n) if deg[v] > 0 and adj[off[v]] < v))
    assert c["finish_vertices"] <= c["worklist"] == int((deg > 2).sum())
    assert c["contract_roots"] == 0
    # contracted link: one compact slot per non-isolated root of the round-0 forest
    ctr.zero_()
    cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(counters=ctr, flags=cc.FLAG_CONTRACT))
    c = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
    assert c["contract_roots"] == int(sum(1 for v in range(n) if deg[v] > 0 and adj[off[v]] >= v))
    assert np.array_equal(u32(lab), oracle.cc_bfs(off, adj))
    assert t.total_ms > 0
    assert np.array_equal(u32(lab), oracle.cc_bfs(off, adj))


def test_microbenchmarks():
    off, adj = gen.rmat(seed=16, scale=11)
    n = off.size - 1
    d_off, d_adj = to_dev(off, adj)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    cc.map_edges(d_off, d_adj, n, out)
    assert np.array_equal(u32(out), np.diff(off).astype(np.uint32))
    x = np.random.default_rng(0).integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    dx = torch.from_numpy(x.view(np.int32)).cuda()
    cc.gather_edges(d_off, d_adj, n, dx, out)
    src = np.repeat(np.arange(n), np.diff(off))
    want = np.zeros(n, dtype=np.uint64)
    np.add.at(want, src, x[adj].astype(np.uint64))
    assert np.array_equal(u32(out), (want & 0xFFFFFFFF).astype(np.uint32))
    s = torch.zeros(1, dtype=torch.int32, device="cuda")
    cc.random_gather(dx, n, 10000, 3, s)
    idx = ((oracle.splitmix64(np.arange(10000, dtype=np.uint64) + np.uint64(3)) & np.uint64(0xFFFFFFFF))
           * np.uint64(n)) >> np.uint64(32)
    assert int(u32(s)[0]) == int(x[idx.astype(np.int64)].astype(np.uint64).sum() & 0xFFFFFFFF)
    dst = torch.empty_like(dx)
    cc.copy(dx, dst, n - n % 4)
    assert torch.equal(dst[: n - n % 4], dx[: n - n % 4])


@pytest.mark.parametrize("samples", [1, 7, 100, 1024, 2048])
def test_identify_frequent_sample_counts(samples):
    off, adj = gen.rmat(seed=17, scale=11)
    n = off.size - 1
    d_off, d_adj = to_dev(off, adj)
    sampled = torch.empty(n, dtype=torch.int32, device="cuda")
    lmax = torch.empty(1, dtype=torch.int32, device="cuda")
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(samples=samples, seed=3, sampled_out=sampled,
                                                              lmax_out=lmax))
    assert int(u32(lmax)[0]) == oracle.identify_frequent(u32(sampled), samples, 3)
    assert np.array_equal(u32(lab), oracle.cc_bfs(off, adj))
    with pytest.raises(cc.CCError):
        cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(samples=2049))


def test_pinned_host_buffers_zero_copy():
    """Pinned host arrays are used in place (zero-copy): same bytes as the device path."""
    off, adj = gen.rmat(seed=18, scale=13)
    n = off.size - 1
    h_off = torch.from_numpy(off).pin_memory()
    h_adj = torch.from_numpy(adj.view(np.int32)).pin_memory()
    h_lab = torch.empty(n, dtype=torch.int32).pin_memory()
    for k in (0, 1, 2):
        cc.cc_labels(h_off, h_adj, n, adj.size, h_lab, cc.make_opts(k=k))
        assert np.array_equal(h_lab.numpy().view(np.uint32), oracle.cc_bfs(off, adj)), k
    h_edges = torch.empty((n, 2), dtype=torch.int32).pin_memory()
    h_ne = torch.zeros(1, dtype=torch.int64).pin_memory()
    cc.cc_spanning_forest(h_off, h_adj, n, adj.size, h_edges, h_ne, h_lab, cc.make_opts())
    want = oracle.cc_bfs(off, adj)
    c = int(np.sum(want == np.arange(n)))
    assert int(h_ne[0]) == n - c
    assert oracle.forest_check(off, adj, c, h_edges[: int(h_ne[0])].numpy().view(np.uint32))[0] == 0
    assert np.array_equal(h_lab.numpy().view(np.uint32), want)
    # mixed: device offsets, pinned adjacency, device labels
    d_off = torch.from_numpy(off).cuda()
    d_lab = torch.empty(n, dtype=torch.int32, device="cuda")
    cc.cc_labels(d_off, h_adj, n, adj.size, d_lab, cc.make_opts())
    assert np.array_equal(u32(d_lab), want)


def test_adversarial_long_chains():
    """Id-ordered paths make round 0 one chain of length n (P[u] = u - 1); the
    compress and finish walks halve paths, so this stays fast and exact."""
    import time
    n = 1 << 21
    ids = np.arange(n - 1, dtype=np.uint64)
    for pairs in (np.stack([ids, ids + 1], 1), np.stack([ids[:-1], ids[:-1] + 2], 1)):
        off, adj = oracle.csr_from_pairs(n, pairs)
        want = oracle.cc_bfs(off, adj)
        for opt in (OPTION_GRID[0], OPTION_GRID[1], dict(k=2, variant="afforest", flags=cc.FLAG_NO_MIDCOMPRESS)):
            t0 = time.time()
            got = run_labels(off, adj, **opt)
            assert time.time() - t0 < 5.0, opt
            assert np.array_equal(got, want), opt


def test_golden_fixtures_gpu():
    """tests/golden/ (paper-cited): cc_labels gives the fixed labels for every k / variant /
    finish, cc_spanning_forest exactly n - c valid edges, and the incremental path inserting
    the edges one batch at a time ends with the same labels."""
    from tests.helpers import golden_fixtures
    for name, off, adj, want in golden_fixtures():
        n = off.size - 1
        for opt in OPTION_GRID[:12]:
            assert np.array_equal(run_labels(off, adj, **opt), want["labels"]), (name, opt)
        d_off, d_adj = to_dev(off, adj)
        edges, lab2 = pkg.spanning_forest(d_off, d_adj)
        E = u32(edges).reshape(-1, 2)
        assert E.shape[0] == want["forest_edges"], name
        assert oracle.forest_check(off, adj, want["components"], E)[0] == 0, name
        assert np.array_equal(u32(lab2), want["labels"]), name
        src = np.repeat(np.arange(n), np.diff(off))
        pairs = np.stack([src, adj.astype(np.int64)], 1)[src < adj].astype(np.int32)
        inc = pkg.IncrementalCC(n)
        for p in pairs:
            inc.batch(torch.from_numpy(p.reshape(1, 2)).cuda(), torch.zeros((0, 2), dtype=torch.int32, device="cuda"))
        assert np.array_equal(u32(inc.labels()), want["labels"]), name
        inc.close()


# ---------------------------------------------------------------------------
def _huge_graphs():
    """Lists longer than kHugeDeg = 2^20 entries (the all-CTA slice bin of the
    finish, cc_static.cu k_finish_big pass 1), P:4091-4100 over hub lists.
    star: one centre (id 3) with 2^20 + 50 leaves, plus a few isolated ids.
    two_hubs: hub 5 with 1.2M leaves and hub 7 with 1.3M leaves (the larger,
    sampled L_max component at k = 1), joined only through vertex x, which is
    the LAST entry of hub 5's list and adjacent to both hubs; and an extra
    path 0-1-2 attached to hub 5's leaf 10 (so the final labels are 0)."""
    n = (1 << 20) + 60
    star = [(3, i) for i in range(4, n - 6)]
    G = [("star", *oracle.csr_from_pairs(n, np.array(star, dtype=np.uint64)))]
    a0, a1 = 10, 10 + 1_200_000
    b0, b1 = a1, a1 + 1_300_000
    x = b1 + 5
    pairs = [(5, i) for i in range(a0, a1)] + [(7, i) for i in range(b0, b1)]
    pairs += [(5, x), (7, x), (0, 1), (1, 2), (2, a0)]
    G.append(("two_hubs", *oracle.csr_from_pairs(x + 3, np.array(pairs, dtype=np.uint64))))
    return G


@pytest.mark.parametrize("opt", [dict(k=0), dict(k=1), dict(k=1, flags=cc.FLAG_NO_SKIP), dict(k=2),
                                 dict(k=0, flags=cc.FLAG_UF_ASYNC), dict(k=1, variant="hybrid", seed=3),
                                 dict(k=0, flags=cc.FLAG_FINISH_SV), dict(k=1, flags=cc.FLAG_FINISH_CRFA),
                                 dict(k=1, flags=cc.FLAG_FINISH_SV), dict(k=0, flags=cc.FLAG_FINISH_CRFA)],
                         ids=lambda o: "-".join(f"{k}{v}" for k, v in o.items()))
def test_huge_list_bin_labels_and_forest(opt):
    """>2^20-entry lists: labels bit-exact and forests valid for k in {0, 1} (the
    'No Sampling' regime of Table 3) and with the skip off.  With the SV /
    CRFA finishes the hub lists are materialised in pieces of 4096 entries by other warps
    (k_sv_pieces), through the filtered (k = 0) and the positioned (k = 1) copy."""
    for name, off, adj in _huge_graphs():
        n = off.size - 1
        assert int(np.diff(off).max()) > (1 << 20) + 1, name
        want = oracle.cc_bfs(off, adj)
        c = int(np.sum(want == np.arange(n)))
        d_off, d_adj = to_dev(off, adj)
        ctr = torch.zeros(len(cc.COUNTER_FIELDS), dtype=torch.int64, device="cuda")
        lab = pkg.connected_components(d_off, d_adj, counters=ctr, **opt)
        assert np.array_equal(u32(lab), want), (name, opt)
        edges, lab2 = pkg.spanning_forest(d_off, d_adj, **opt)
        rc, bad = oracle.forest_check(off, adj, c, u32(edges).reshape(-1, 2))
        assert rc == 0, (name, opt, oracle.FOREST_ERRORS[rc], bad)
        assert np.array_equal(u32(lab2), want), (name, opt)
        cnt = dict(zip(cc.COUNTER_FIELDS, ctr.cpu().tolist()))
        sv = opt.get("flags", 0) & (cc.FLAG_FINISH_SV | cc.FLAG_FINISH_CRFA)
        if not sv and (opt["k"] == 0 or opt.get("flags") == cc.FLAG_NO_SKIP or (name == "two_hubs" and opt["k"] == 1)):
            # the hub list went through the finish (the huge bin) -- not skipped
            assert cnt["finish_edges"] > (1 << 20), (name, opt, cnt["finish_edges"])


def test_cuda_graph_capture_replay():
    """cc_labels with device buffers is stream-ordered with no host synchronisation, so a
    caller can capture it into a CUDA graph (kernels, stream-ordered scratch allocations,
    programmatic-dependent launches) and replay it -- the launch-bound small configs (C1)
    then pay one graph launch per call.  Replays must give the same labels."""
    off, adj = gen.er(seed=1)                       # C1's recipe
    n = off.size - 1
    want = oracle.cc_bfs(off, adj)
    d_off, d_adj = to_dev(off, adj)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(), s)      # warm-up outside capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        cc.cc_labels(d_off, d_adj, n, adj.size, lab, cc.make_opts(), s)
    for _ in range(5):
        lab.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(u32(lab), want)
