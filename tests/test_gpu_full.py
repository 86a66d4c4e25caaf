"""Full-size BASELINE.json configs (C1-C5), in the launch configuration bench.py times.

The graphs come from the CUDA generator (byte-identical to inputs/gen.py, see
test_gpu_gen.py); the oracle runs on the host over the same bytes.  Labels and
answers are compared element by element (bit-exact); forests by the validity
triple.  These are minutes-long on one B200 + its host cores."""
import time

import numpy as np
import pytest

import inputs
import oracle
from tests.helpers import u32

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2008_03909_b200 as pkg  # noqa: E402
from inputs import gpu as ggen  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402


def host(t, dtype):
    return t.cpu().numpy().view(dtype)


_GRAPHS = {}


def full_graph(cfg):
    """(device off, device adj, host off, host adj, oracle labels, #components), built once
    per config and module (the C4 oracle BFS alone takes ~30 s on one host core)."""
    if cfg.name not in _GRAPHS:
        _GRAPHS.clear()                                  # one full-size graph resident at a time
        torch.cuda.empty_cache()
        d_off, d_adj = ggen.config_graph(cfg)
        off = host(d_off, np.int64)
        adj = host(d_adj, np.uint32)
        t0 = time.time()
        want = oracle.cc_bfs(off, adj)
        print(f"{cfg.name}: oracle {time.time() - t0:.1f}s")
        c = int(np.sum(want == np.arange(off.size - 1)))
        _GRAPHS[cfg.name] = (d_off, d_adj, off, adj, want, c)
    return _GRAPHS[cfg.name]


def check_static(cfg, **opt):
    d_off, d_adj, off, adj, want, c = full_graph(cfg)
    t0 = time.time()
    lab = pkg.connected_components(d_off, d_adj, **opt)
    got = u32(lab)
    del lab
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (cfg.name, opt, bad[:5], got[bad[:5]], want[bad[:5]])
    edges, lab2 = pkg.spanning_forest(d_off, d_adj, **opt)
    E = u32(edges)
    got2 = u32(lab2)
    del edges, lab2
    assert np.array_equal(got2, want), (cfg.name, opt)
    rc, idx = oracle.forest_check(off, adj, c, E)
    assert rc == 0, (cfg.name, opt, oracle.FOREST_ERRORS[rc], idx)
    print(f"{cfg.name} {opt}: n={off.size - 1} m={adj.size} components={c} gpu {time.time() - t0:.1f}s")


@pytest.mark.parametrize("cfg", [inputs.C1, inputs.C2, inputs.C3, inputs.C4], ids=lambda c: c.name)
def test_static_config_bit_exact(cfg):
    """Default options (afforest k = 2), the launch configuration bench.py times."""
    check_static(cfg)


@pytest.mark.parametrize("opt", [dict(k=0), dict(k=2, variant="hybrid", seed=4),
                                 dict(k=0, flags=1 << 9), dict(k=0, flags=1 << 13)],
                         ids=["k0", "hybrid-k2", "k0-sv", "k0-crfa"])
def test_c4_no_sampling_and_hybrid(opt):
    """SURVEY 8(c) test matrix, C4 column: k in {0, 2}.  k = 0 is Table 3's 'No Sampling'
    regime: every one of the 4.2e9 entries goes through the finish meta-loop
    (P:4091-4100), hub lists of > 2^20 entries through the all-CTA bin; hybrid k = 2 is the
    paper's default sampling.  The NEXT-3 finishes (Shiloach-Vishkin,
    CC_FLAG_FINISH_SV = 1 << 9; Liu-Tarjan CRFA, CC_FLAG_FINISH_CRFA = 1 << 13) run here on
    every edge too, in the configuration profiles/r2_next3_sv_crfa.json times.  Labels
    bit-exact, forest validity triple."""
    check_static(inputs.C4, **opt)


def test_incremental_config_multi_batch_call_bit_exact():
    """C5 in the launch configuration bench.py times: the whole 256-batch stream in ONE
    cc_incr_batches call on device-resident pairs (kernels after the first read their pairs
    and first parents before their PDL wait).  Every answer and the final labels == oracle."""
    _GRAPHS.clear()
    torch.cuda.empty_cache()
    cfg = inputs.C5
    n = 1 << cfg.scale
    nb = cfg.n_batches
    ins = torch.empty((nb, cfg.n_ins, 2), dtype=torch.int32, device="cuda")
    qs = torch.empty((nb, cfg.n_q, 2), dtype=torch.int32, device="cuda")
    for b in range(nb):
        ggen.incr_batch(cfg.seed, cfg.scale, b, cfg.n_ins, cfg.n_q, ins[b], qs[b])
    ans = torch.empty((nb, cfg.n_q), dtype=torch.uint8, device="cuda")
    h = cc.Incr(n)
    h.batches(np.full(nb, cfg.n_ins, dtype=np.int64), ins, np.full(nb, cfg.n_q, dtype=np.int64), qs, ans)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab)
    h.close()
    h_ins, h_qs = host(ins, np.uint32), host(qs, np.uint32)
    del ins, qs
    want, want_lab = oracle.incr_run(n, [(h_ins[b], h_qs[b]) for b in range(nb)], want_labels=True)
    got = ans.cpu().numpy().reshape(-1)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, bad[:5]
    assert np.array_equal(u32(lab), want_lab)


def test_incremental_config_bit_exact():
    _GRAPHS.clear()                       # release the full-size static graph (device + host)
    torch.cuda.empty_cache()
    cfg = inputs.C5
    n = 1 << cfg.scale
    inc = pkg.IncrementalCC(n)
    ins = torch.empty((cfg.n_ins, 2), dtype=torch.int32, device="cuda")
    qs = torch.empty((cfg.n_q, 2), dtype=torch.int32, device="cuda")
    answers, h_ins, h_qs = [], [], []
    for b in range(cfg.n_batches):
        ggen.incr_batch(cfg.seed, cfg.scale, b, cfg.n_ins, cfg.n_q, ins, qs)
        a = inc.batch(ins, qs)
        answers.append(a.cpu().numpy())
        h_ins.append(host(ins, np.uint32).copy())
        h_qs.append(host(qs, np.uint32).copy())
    lab = u32(inc.labels())
    inc.close()
    got = np.concatenate(answers)
    want, want_lab = oracle.incr_run(n, list(zip(h_ins, h_qs)), want_labels=True)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, bad[:5]
    assert np.array_equal(lab, want_lab)
    print(f"C5: {got.size} answers, {int(want.sum())} true")


def test_amsf_c3_bucket_counts():
    """NEXT-4 at C3 size (RMAT-24, Exp(1) weights from the CUDA generator, eps =
    0.25): a valid spanning forest whose per-bucket edge counts equal the oracle's
    (which, with every weight inside its bucket, implies the (1+eps) sandwich)."""
    cfg = inputs.C3
    d_off, d_adj = ggen.config_graph(cfg)
    d_w = ggen.exp_weights(d_off, d_adj, cfg.seed)
    E, W, tot = pkg.amsf(d_off, d_adj, d_w, 0.25)
    torch.cuda.synchronize()
    E = u32(E).reshape(-1, 2)
    W = W.cpu().numpy()
    off = host(d_off, np.int64)
    adj = host(d_adj, np.uint32)
    w = d_w.cpu().numpy()
    del d_off, d_adj, d_w
    torch.cuda.empty_cache()
    n = off.size - 1
    lab = oracle.cc_bfs(off, adj)
    c = int(np.sum(lab == np.arange(n)))
    rc, idx = oracle.forest_check(off, adj, c, E)
    assert rc == 0, (oracle.FOREST_ERRORS[rc], idx)
    want = oracle.amsf(off, adj, w, 0.25)
    b = oracle.amsf_bounds(w.min(), w.max(), 0.25)
    assert np.array_equal(np.bincount(oracle.amsf_bucket(W, b), minlength=want["nbuckets"]),
                          np.bincount(want["buckets"], minlength=want["nbuckets"]))
    assert tot == pytest.approx(float(W.astype(np.float64).sum()), rel=1e-12)
    print(f"C3 AMSF: n={n} forest={E.shape[0]} W={tot:.6g} oracle W={want['total']:.6g} buckets={want['nbuckets']}")


def test_maximum_n_labels_and_forest():
    """n = 0xFFFFFFFE, the largest the ABI accepts (uint32 ids, 0xFFFFFFFF is the
    sentinel): every grid, tile tail and 32/64-bit index path at its limit.
    A few edges join vertices at both ends of the id range; everything else is
    isolated.  (34 GB offsets + 17 GB labels + scratch, on one B200.)"""
    n = 0xFFFFFFFE
    pairs = [(0, n - 1), (n - 1, 1 << 31), (1 << 31, (1 << 31) + 1), ((1 << 31) + 1, 12345), (n - 2, n - 3),
             (1 << 32 - 2, 7)]
    adjl = {}
    for a, b in pairs:
        adjl.setdefault(a, []).append(b)
        adjl.setdefault(b, []).append(a)
    verts = sorted(adjl)
    adj = np.array([x for v in verts for x in sorted(adjl[v])], dtype=np.uint32)
    off = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    acc = 0
    for v in verts:                                       # off[v+1:] += deg(v), as a step function
        acc_next = acc + len(adjl[v])
        off[v + 1:] += len(adjl[v])
        acc = acc_next
    d_adj = torch.from_numpy(adj.view(np.int32)).cuda()
    lab = pkg.connected_components(off, d_adj)
    torch.cuda.synchronize()
    # expected: min id per component
    comp = {}
    par = {v: v for v in verts}

    def find(x):
        while par[x] != x:
            x = par[x]
        return x
    for a, b in pairs:
        ra, rb = find(a), find(b)
        if ra != rb:
            par[max(ra, rb)] = min(ra, rb)
    for v in verts:
        comp[v] = find(v)
    got = {v: int(np.uint32(lab[v].item() & 0xFFFFFFFF)) for v in verts}
    assert got == comp, (got, comp)
    # everything else is its own label: count the non-identity slots chunk by chunk
    moved = 0
    step = 1 << 30
    for s0 in range(0, n, step):
        s1 = min(n, s0 + step)
        ids = torch.arange(s0, s1, dtype=torch.int64, device="cuda")
        moved += int(((lab[s0:s1].to(torch.int64) & 0xFFFFFFFF) != ids).sum().item())
        del ids
    assert moved == sum(1 for v in verts if comp[v] != v)
    del lab
    torch.cuda.empty_cache()
    edges, lab2 = pkg.spanning_forest(off, d_adj, with_labels=False)
    E = u32(edges).reshape(-1, 2)
    assert E.shape[0] == sum(1 for v in verts if comp[v] != v)
    for a, b in E.tolist():
        assert b in adjl[a] and find(a) == find(b)


def test_more_than_2_32_adjacency_entries():
    """m > 2^32 (64-bit adjacency indexing everywhere): 256 disjoint cliques of 4101
    vertices, 4,304,409,600 entries (17.2 GB); every list exceeds the CTA-per-list
    threshold, so the finish's long-list path is exercised too.  Labels must be the
    first vertex of each clique."""
    B, nb = 4101, 256
    n = B * nb
    d = B - 1
    m = n * d
    assert m > (1 << 32)
    off = torch.arange(0, n + 1, dtype=torch.int64, device="cuda") * d
    adj = torch.empty(m, dtype=torch.int32, device="cuda")
    j = torch.arange(d, dtype=torch.int64, device="cuda")
    step = 8192
    for v0 in range(0, n, step):
        v = torch.arange(v0, min(n, v0 + step), dtype=torch.int64, device="cuda")
        b = (v // B) * B
        r = (v - b).unsqueeze(1)
        vals = b.unsqueeze(1) + j.unsqueeze(0) + (j.unsqueeze(0) >= r).to(torch.int64)
        adj[v0 * d:(v0 + v.numel()) * d] = vals.reshape(-1).to(torch.int32)
        del vals
    torch.cuda.synchronize()
    want = (torch.arange(n, device="cuda", dtype=torch.int64) // B) * B
    for kw in (dict(), dict(k=0)):
        lab = pkg.connected_components(off, adj, **kw)
        torch.cuda.synchronize()
        assert torch.equal(lab.to(torch.int64), want), kw
    del adj
    torch.cuda.empty_cache()
