"""Seeded input generators (inputs/gen.py): validity, determinism, statistics."""
import numpy as np
import pytest

from inputs import gen


@pytest.mark.parametrize("s", [1, 2, 3, 5, 8, 13, 20])
def test_permutation_is_bijective(s):
    x = np.arange(1 << s, dtype=np.uint64)
    y = gen.permute(x, seed=4, s=s)
    assert np.array_equal(np.sort(y), x)
    if s >= 8:
        assert not np.array_equal(y, x)


def test_csr_valid_and_deterministic():
    for make in (lambda sd: gen.er(seed=sd), lambda sd: gen.grid(seed=sd, rows=128, cols=96),
                 lambda sd: gen.rmat(seed=sd, scale=12)):
        off, adj = make(1)
        gen.validate_csr(off, adj)
        off2, adj2 = make(1)
        assert np.array_equal(off, off2) and np.array_equal(adj, adj2)
        off3, adj3 = make(2)
        assert not (off3.size == off.size and np.array_equal(off3, off) and np.array_equal(adj3, adj))


def test_validate_csr_rejects_defects():
    off, adj = gen.rmat(seed=3, scale=8)
    gen.validate_csr(off, adj)
    bad = adj.copy()
    bad[[0, 1]] = bad[[1, 0]]                       # unsorted
    with pytest.raises(AssertionError):
        gen.validate_csr(off, bad)
    off2 = off.copy()
    off2[5] += 1                                    # breaks symmetry / sortedness
    with pytest.raises(AssertionError):
        gen.validate_csr(off2, adj)


def test_er_c1_shape():
    off, adj = gen.er()
    n = off.size - 1
    assert n == 101_000
    assert np.all(np.diff(off)[100_000:] == 0)       # 1,000 appended isolated vertices
    # E[self-loops] = 4, E[dup pairs] ~ 16: m = 2 * (400000 - drops), drops small
    assert 2 * (400_000 - 200) <= adj.size <= 2 * 400_000
    assert adj.size % 2 == 0


def test_grid_edge_count_within_5_sigma():
    R = C = 512
    off, adj = gen.grid(seed=2, rows=R, cols=C)
    cand = R * (C - 1) + (R - 1) * C
    p = gen.P55 / 2 ** 32
    mu, sd = cand * p, np.sqrt(cand * p * (1 - p))
    assert abs(adj.size / 2 - mu) < 5 * sd
    # every kept edge is a lattice edge
    src = np.repeat(np.arange(R * C), np.diff(off))
    d = np.abs(src - adj.astype(np.int64))
    assert np.all((d == 1) | (d == C))
    assert np.all((d != 1) | (np.minimum(src, adj) % C != C - 1))   # no wrap-around


def test_rmat_quadrant_frequencies():
    # unpermuted, level-0 bits give the quadrant of each draw: (a, b, c, d) = (.57, .19, .19, .05)
    s = 10
    u, v = gen.rmat_pairs(seed=3, s=s, first=0, count=200_000, permuted=False)
    top_u = (u >> np.uint64(s - 1)) & np.uint64(1)
    top_v = (v >> np.uint64(s - 1)) & np.uint64(1)
    q = (top_u * np.uint64(2) + top_v).astype(np.int64)
    freq = np.bincount(q, minlength=4) / q.size
    for f, p in zip(freq, (0.57, 0.19, 0.19, 0.05)):
        assert abs(f - p) < 5 * np.sqrt(p * (1 - p) / q.size)


def test_incr_batch_shapes():
    ins, qs = gen.incr_batch(seed=5, scale=12, b=3, n_ins=1000, n_q=100)
    assert ins.shape == (1000, 2) and qs.shape == (100, 2)
    assert ins.max() < 4096 and qs.max() < 4096
    # draws are indexed globally: batch b covers draws b*n_ins .. (b+1)*n_ins-1
    u, v = gen.rmat_pairs(5, 12, 3000, 1000)
    assert np.array_equal(ins[:, 0], u.astype(np.uint32)) and np.array_equal(ins[:, 1], v.astype(np.uint32))
