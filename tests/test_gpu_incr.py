"""GPU parity of the batch-incremental path (cc_incr_*) vs the sequential DSU oracle.

Answers must be bit-exact (reading R15: a query sees all inserts of its own
batch).  cc_incr_labels after the stream must equal the static oracle on the
union of the inserts (cross-pins the static and incremental paths)."""
import numpy as np
import pytest

import oracle
from inputs import gen
from tests.helpers import u32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2008_03909_b200 as pkg  # noqa: E402
from paper_2008_03909_b200 import cc  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32).reshape(-1, 2)).cuda()


def run_stream(n, batches, flags=0):
    inc = pkg.IncrementalCC(n, flags=flags)
    outs = []
    for ins, qs in batches:
        a = inc.batch(dev(ins), dev(qs))
        outs.append(a.cpu().numpy())
    lab = u32(inc.labels())
    inc.close()
    return np.concatenate(outs) if outs else np.zeros(0, np.uint8), lab


def static_labels(n, batches):
    pairs = np.concatenate([np.asarray(b[0], dtype=np.uint32).reshape(-1, 2) for b in batches])
    off, adj = oracle.csr_from_pairs(n, pairs)
    return oracle.cc_bfs(off, adj)


@pytest.mark.parametrize("flags", [0, cc.FLAG_HALVE, cc.FLAG_UF_ASYNC, cc.FLAG_FIND_SPLIT, cc.FLAG_FIND_NAIVE])
@pytest.mark.parametrize("batch", [1, 10, 256, 257, 1000, 1 << 14])
def test_stream_bit_exact(flags, batch):
    scale = 12
    n = 1 << scale
    total = 3 * (1 << 14) if batch >= 1000 else 400
    n_ins = max(1, int(batch * 0.9))
    n_q = max(1, batch - n_ins)
    nb = max(1, total // batch)
    batches = [gen.incr_batch(seed=5, scale=scale, b=b, n_ins=n_ins, n_q=n_q) for b in range(nb)]
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    got, lab = run_stream(n, batches, flags)
    assert np.array_equal(got, want), (flags, batch, np.nonzero(got != want)[0][:5])
    assert np.array_equal(lab, want_lab)
    assert np.array_equal(lab, static_labels(n, batches))


def test_true_heavy_stream():
    """Half the queries are endpoints of earlier inserts (guaranteed 1), half join
    random vertices of the current giant -- catches an 'always 0' bug."""
    rng = np.random.default_rng(4)
    n = 1 << 13
    batches = []
    prev = np.zeros((0, 2), dtype=np.uint32)
    for b in range(40):
        ins, _ = gen.incr_batch(seed=6, scale=13, b=b, n_ins=2000, n_q=1)
        pool = np.concatenate([prev, ins])
        pick = pool[rng.integers(0, pool.shape[0], 300)]
        mixed = np.stack([pick[:, 0], pool[rng.integers(0, pool.shape[0], 300), 1]], 1)
        qs = np.concatenate([pick, mixed, rng.integers(0, n, (50, 2)).astype(np.uint32)])
        batches.append((ins, qs))
        prev = pool
    want, _ = oracle.incr_run(n, batches)
    got, _ = run_stream(n, batches)
    assert np.array_equal(got, want)
    assert want.mean() > 0.5


def test_closed_forms_and_monotone():
    n = 64
    batches = [
        (np.array([[0, 1], [1, 2]]), np.array([[0, 2], [3, 3], [0, 3]])),
        (np.array([[2, 3], [5, 5], [5, 5]]), np.array([[0, 3], [5, 9], [3, 0], [5, 5]])),
        (np.zeros((0, 2), int), np.array([[0, 2], [0, 3], [63, 63], [62, 63]])),
        (np.array([[62, 63]]), np.zeros((0, 2), int)),
        (np.zeros((0, 2), int), np.array([[62, 63]])),
    ]
    got, lab = run_stream(n, batches)
    assert got.tolist() == [1, 1, 0, 1, 0, 1, 1, 1, 1, 1, 0, 1]
    assert lab[3] == 0 and lab[63] == 62


def test_validate_and_errors():
    inc = pkg.IncrementalCC(100, flags=cc.FLAG_VALIDATE)
    with pytest.raises(cc.CCError):
        inc.batch(dev([[1, 2], [3, 100]]), dev([[0, 1]]))
    # the failed batch applied nothing
    a = inc.batch(dev([[5, 6]]), dev([[1, 2], [5, 6]]))
    assert a.cpu().tolist() == [0, 1]
    inc.close()


def test_host_buffers():
    n = 1 << 10
    batches = [gen.incr_batch(seed=8, scale=10, b=b, n_ins=300, n_q=100) for b in range(5)]
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    h = cc.Incr(n)
    outs = []
    for ins, qs in batches:
        ans = np.zeros(qs.shape[0], dtype=np.uint8)
        h.batch(np.ascontiguousarray(ins), ins.shape[0], np.ascontiguousarray(qs), qs.shape[0], ans)
        outs.append(ans)
    lab = np.zeros(n, dtype=np.uint32)
    h.labels(lab)
    h.close()
    assert np.array_equal(np.concatenate(outs), want)
    assert np.array_equal(lab, want_lab)


def test_pinned_host_buffers_zero_copy():
    n = 1 << 11
    batches = [gen.incr_batch(seed=9, scale=11, b=b, n_ins=500, n_q=200) for b in range(4)]
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    h = cc.Incr(n)
    outs = []
    for ins, qs in batches:
        ti = torch.from_numpy(ins.view(np.int32)).pin_memory()
        tq = torch.from_numpy(qs.view(np.int32)).pin_memory()
        ta = torch.zeros(qs.shape[0], dtype=torch.uint8).pin_memory()
        h.batch(ti, ins.shape[0], tq, qs.shape[0], ta)
        outs.append(ta.numpy().copy())
    lab = torch.empty(n, dtype=torch.int32).pin_memory()
    h.labels(lab)
    h.close()
    assert np.array_equal(np.concatenate(outs), want)
    assert np.array_equal(lab.numpy().view(np.uint32), want_lab)


@pytest.mark.parametrize("flags", [cc.FLAG_WAIT_FREE, cc.FLAG_WAIT_FREE | cc.FLAG_HALVE,
                                   cc.FLAG_WAIT_FREE | cc.FLAG_UF_ASYNC])
def test_wait_free_prefix_soundness(flags):
    """Type (1): inserts and queries of a batch run concurrently.  Answers
    are linearizable: 1 => connected after batches 0..i, 0 => not connected after
    batches 0..i-1; final labels are still exact."""
    scale = 12
    n = 1 << scale
    batches = [gen.incr_batch(seed=12, scale=scale, b=b, n_ins=3000, n_q=3000) for b in range(12)]
    after, want_lab = oracle.incr_run(n, batches, want_labels=True)
    empty = np.zeros((0, 2), np.uint32)
    before_batches = [(batches[i - 1][0] if i else empty, batches[i][1]) for i in range(len(batches))]
    before, _ = oracle.incr_run(n, before_batches)
    got, lab = run_stream(n, batches, flags)
    assert np.all(got[got == 1] <= after[got == 1])      # 1 => connected after the batch
    assert np.all(before[got == 0] == 0)                 # 0 => not connected before it
    assert np.array_equal(lab, want_lab)
    # the contract has room: answers that changed inside a batch are either value
    undecided = (after == 1) & (before == 0)
    assert np.array_equal(got[~undecided], after[~undecided])


@pytest.mark.parametrize("batch", [1, 10, 1000, 9000])
@pytest.mark.parametrize("flags", [0, cc.FLAG_FIND_SPLIT | cc.FLAG_HALVE, cc.FLAG_VALIDATE, cc.FLAG_FIND_NAIVE])
def test_multi_batch_call_bit_exact(batch, flags):
    """cc_incr_batches == a sequence of cc_incr_batch calls == the oracle."""
    n = 1 << 12
    nb = max(1, 20000 // batch)
    n_ins = max(1, int(batch * 0.9))
    n_q = max(1, batch - n_ins)
    batches = [gen.incr_batch(seed=14, scale=12, b=b, n_ins=n_ins, n_q=n_q) for b in range(nb)]
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    ins = dev(np.concatenate([b[0] for b in batches]))
    qs = dev(np.concatenate([b[1] for b in batches]))
    ans = torch.empty(qs.shape[0], dtype=torch.uint8, device="cuda")
    h = cc.Incr(n, flags)
    h.batches(np.full(nb, n_ins), ins, np.full(nb, n_q), qs, ans)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab)
    h.close()
    assert np.array_equal(ans.cpu().numpy(), want)
    assert np.array_equal(u32(lab), want_lab)


@pytest.mark.parametrize("flags", [0, cc.FLAG_HALVE, cc.FLAG_FIND_SPLIT])
def test_multi_batch_call_large_batches_mixed_shapes(flags):
    """cc_incr_batches with batches above the single-CTA limit (two kernels per batch, the
    pre-wait pair / first-parent reads after the first kernel): an empty then a queries-only
    first batch, inserts-only batches, empty batches and uneven sizes; answers and labels ==
    oracle."""
    n = 1 << 14
    rng = np.random.default_rng(5)
    shapes = [(0, 0), (0, 9000), (12000, 0), (0, 0), (20000, 3000), (9001, 1), (1, 9001), (30000, 30000), (0, 0),
              (15000, 5000)]
    batches = []
    for b, (ni, nq) in enumerate(shapes):
        i, _ = gen.incr_batch(seed=21, scale=14, b=b, n_ins=max(ni, 1), n_q=1)
        q = rng.integers(0, n, (nq, 2)).astype(np.uint32)
        batches.append((i[:ni], q))
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    ins = dev(np.concatenate([b[0] for b in batches]).reshape(-1, 2))
    qs = dev(np.concatenate([b[1] for b in batches]).reshape(-1, 2))
    ans = torch.empty(qs.shape[0], dtype=torch.uint8, device="cuda")
    h = cc.Incr(n, flags)
    h.batches(np.array([s[0] for s in shapes]), ins, np.array([s[1] for s in shapes]), qs, ans)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab)
    h.close()
    assert np.array_equal(ans.cpu().numpy(), want)
    assert np.array_equal(u32(lab), want_lab)


def test_adversarial_chain_queries():
    """A path inserted in id order builds one chain of length n (every hook puts
    i+1 under i); the default halving queries must answer it exactly and fast,
    in one batch and in many small batches (the single-CTA path)."""
    import time
    n = 1 << 20
    ids = np.arange(n - 1, dtype=np.uint32)
    path = np.stack([ids, ids + 1], 1)
    rng = np.random.default_rng(4)
    qs = rng.integers(0, n, (1 << 16, 2)).astype(np.uint32)
    qs[:100, 1] = qs[:100, 0]
    want, _ = oracle.incr_run(n, [(path, qs)])
    for flags in (0, cc.FLAG_FIND_SPLIT):
        inc = pkg.IncrementalCC(n, flags=flags)
        t0 = time.time()
        ans = inc.batch(torch.from_numpy(path.view(np.int32)).cuda(), torch.from_numpy(qs.view(np.int32)).cuda())
        torch.cuda.synchronize()
        assert time.time() - t0 < 5.0
        assert np.array_equal(ans.cpu().numpy(), want)
        inc.close()
    # wait-free: answers are only prefix-sound here (everything connects during the batch);
    # a == b must be 1, and it must stay fast on the chain
    inc = pkg.IncrementalCC(n, flags=cc.FLAG_WAIT_FREE)
    t0 = time.time()
    ans = inc.batch(torch.from_numpy(path.view(np.int32)).cuda(), torch.from_numpy(qs.view(np.int32)).cuda())
    torch.cuda.synchronize()
    assert time.time() - t0 < 5.0
    assert ans.cpu().numpy()[:100].all()
    inc.close()
    # small batches: 256 inserts each, a query batch at the end (k_small_batches)
    inc = pkg.IncrementalCC(4096)
    small = path[:4095]
    batches = [(small[i:i + 256], qs[:64] % 4096) for i in range(0, 4095, 256)]
    want2, _ = oracle.incr_run(4096, batches)
    got = []
    for ins, q in batches:
        got.append(inc.batch(torch.from_numpy(np.ascontiguousarray(ins).view(np.int32)).cuda(),
                             torch.from_numpy(np.ascontiguousarray(q).view(np.int32)).cuda()).cpu().numpy())
    assert np.array_equal(np.concatenate(got), want2)
    inc.close()


@pytest.mark.parametrize("where", ["both_pinned", "ins_pinned", "q_pinned"])
def test_multi_batch_pinned_pipelined(where):
    """cc_incr_batches over pinned HOST batches (the double-buffered DMA staging path):
    ragged batch sizes (incl. empty inserts / queries and batches above the single-CTA
    threshold), answers written to pinned host memory -- bit-exact vs the oracle."""
    n = 1 << 16
    rng = np.random.default_rng(8)
    sizes = [(20000, 3000), (0, 500), (9000, 0), (30000, 7000), (1, 1), (50000, 12000), (17, 9000)]
    batches = []
    for b, (ni, nq) in enumerate(sizes):
        ins, qs = gen.incr_batch(seed=21, scale=16, b=b, n_ins=max(ni, 1), n_q=max(nq, 1))
        batches.append((ins[:ni], qs[:nq]))
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    ins_all = torch.from_numpy(np.concatenate([b[0] for b in batches]).astype(np.uint32).view(np.int32))
    qs_all = torch.from_numpy(np.concatenate([b[1] for b in batches]).astype(np.uint32).view(np.int32))
    ins_arg = ins_all.pin_memory() if where in ("both_pinned", "ins_pinned") else ins_all.cuda()
    qs_arg = qs_all.pin_memory() if where in ("both_pinned", "q_pinned") else qs_all.cuda()
    ans = torch.zeros(qs_all.shape[0], dtype=torch.uint8).pin_memory()
    h = cc.Incr(n)
    h.batches(np.array([s[0] for s in sizes]), ins_arg, np.array([s[1] for s in sizes]), qs_arg, ans)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab)
    h.close()
    assert np.array_equal(ans.numpy(), want)
    assert np.array_equal(u32(lab), want_lab)


def test_multi_batch_pinned_validate():
    """CC_FLAG_VALIDATE on the pinned multi-batch path: ids are checked before any batch
    is staged or applied (an out-of-range id anywhere rejects the whole call)."""
    n = 1 << 12
    batches = [gen.incr_batch(seed=3, scale=12, b=b, n_ins=20000, n_q=500) for b in range(3)]
    ins = np.concatenate([b[0] for b in batches]).astype(np.uint32)
    qs = np.concatenate([b[1] for b in batches]).astype(np.uint32)
    want, want_lab = oracle.incr_run(n, batches, want_labels=True)
    ans = torch.zeros(qs.shape[0], dtype=torch.uint8).pin_memory()
    h = cc.Incr(n, cc.FLAG_VALIDATE)
    h.batches(np.full(3, 20000), torch.from_numpy(ins.view(np.int32)).pin_memory(), np.full(3, 500),
              torch.from_numpy(qs.view(np.int32)).pin_memory(), ans)
    assert np.array_equal(ans.numpy(), want)
    bad = ins.copy()
    bad[-1, 1] = n                                        # last insert of the last batch
    lab0 = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab0)
    with pytest.raises(cc.CCError):
        h.batches(np.full(3, 20000), torch.from_numpy(bad.view(np.int32)).pin_memory(), np.full(3, 500),
                  torch.from_numpy(qs.view(np.int32)).pin_memory(), ans)
    lab1 = torch.empty(n, dtype=torch.int32, device="cuda")
    h.labels(lab1)
    h.close()
    assert torch.equal(lab0, lab1)                        # nothing applied
    assert np.array_equal(u32(lab0), want_lab)


def test_repeat_random_batch_shapes():
    """SURVEY 8(c) test matrix, C5 column "small": repeated streams whose batch sizes, insert /
    query mix and options are random, so every launch path is taken in every order (the one-CTA
    small batch, the two PDL kernels, the multi-batch kernel, validation) -- answers bit-exact."""
    rng = np.random.default_rng(5)
    n = 1 << 13
    flag_pool = [0, cc.FLAG_HALVE, cc.FLAG_UF_ASYNC, cc.FLAG_FIND_SPLIT, cc.FLAG_FIND_NAIVE, cc.FLAG_VALIDATE]
    for it in range(40):
        flags = int(rng.choice(flag_pool))
        nb = int(rng.integers(1, 12))
        batches = []
        for b in range(nb):
            size = int(rng.choice([1, 7, 32, 255, 256, 257, 1000, 5000, 20000]))
            n_q = int(rng.integers(0, size + 1))
            ins, qs = gen.incr_batch(seed=100 + it, scale=13, b=b, n_ins=max(size - n_q, 0), n_q=n_q)
            batches.append((ins, qs))
        want, want_lab = oracle.incr_run(n, batches, want_labels=True)
        if it % 2:
            got, lab = run_stream(n, batches, flags)
        else:                                         # the same batches through one cc_incr_batches call
            h = cc.Incr(n, flags)
            ic = np.array([b[0].size // 2 for b in batches], dtype=np.int64)
            qc = np.array([b[1].size // 2 for b in batches], dtype=np.int64)
            d_ins = dev(np.concatenate([b[0] for b in batches])) if ic.sum() else torch.zeros((0, 2), dtype=torch.int32,
                                                                                                device="cuda")
            d_q = dev(np.concatenate([b[1] for b in batches])) if qc.sum() else torch.zeros((0, 2), dtype=torch.int32,
                                                                                              device="cuda")
            ans = torch.empty(max(int(qc.sum()), 1), dtype=torch.uint8, device="cuda")
            h.batches(ic, d_ins, qc, d_q, ans)
            lab_t = torch.empty(n, dtype=torch.int32, device="cuda")
            h.labels(lab_t)
            torch.cuda.synchronize()
            got, lab = ans.cpu().numpy()[: int(qc.sum())], u32(lab_t)
            h.close()
        assert np.array_equal(got, want), (it, flags, [b[0].size // 2 for b in batches])
        assert np.array_equal(lab, want_lab), it
