"""Seeded synthetic inputs (numpy, CPU) -- no arithmetic of the method lives here.

These generators stand in for the paper's datasets (road_usa, LiveJournal,
Twitter, Friendster, ... P:1145-1175, Table 2), which are not in
the container: the five BASELINE.json configs, with the recipe of DESIGN.md
§Inputs.  Every draw is a pure function of (seed, stream, index) through

    mix(seed, stream, i) = splitmix64(seed * GOLD + stream * 2^40 + i)   (mod 2^64)

so the CUDA generator (``inputs/csrc/gen.cu``) reproduces these bytes exactly,
independent of launch configuration (tested in tests/test_gen_gpu.py).  The
oracle consumes CSRs from here (small sizes) or the GPU generator's bytes
(full sizes, after the byte-equality test at small sizes); the product library
consumes them through device memory.

CSR convention: symmetric, no self-loops, no duplicates,
every list sorted ascending; int64 offsets[n+1], uint32 adj[m], m = number of
directed entries (each undirected edge counted twice).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15

ER_STREAM, GRID_STREAM, RMAT_STREAM, PERM_STREAM, QUERY_STREAM, WEIGHT_STREAM = 1, 2, 3, 4, 5, 6

# fixed-point thresholds: floor(p * 2^32)
P55 = 2362232012            # Bernoulli(0.55) for the grid
RMAT_T1 = 2448131358        # a            = 0.57
RMAT_T2 = 3264175144        # a + b        = 0.76
RMAT_T3 = 4080218931        # a + b + c    = 0.95


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(GOLD)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def mix(seed: int, stream: int, idx) -> np.ndarray:
    base = np.uint64((seed * GOLD + (stream << 40)) & M64)
    with np.errstate(over="ignore"):
        return splitmix64(np.asarray(idx, dtype=np.uint64) + base)


def lo32(r):
    return r & np.uint64(0xFFFFFFFF)


def hi32(r):
    return r >> np.uint64(32)


def scale_u32(x32, bound: int):
    """(x32 * bound) >> 32 : uniform on [0, bound) from a 32-bit draw."""
    with np.errstate(over="ignore"):
        return (x32 * np.uint64(bound)) >> np.uint64(32)


# ---------------------------------------------------------------------------
def perm_params(seed: int, s: int):
    """Three rounds of x ^= x >> ceil(s/2); x = x*K_i + c_i (mod 2^s), K_i odd."""
    mask = (1 << s) - 1
    r = [int(v) for v in mix(seed, PERM_STREAM, np.arange(6, dtype=np.uint64))]
    ks = [(r[i] | 1) & mask for i in range(3)]
    cs = [r[3 + i] & mask for i in range(3)]
    return ks, cs, (s + 1) // 2, mask


def permute(x, seed: int, s: int) -> np.ndarray:
    """Seeded bijection on s-bit ids (Q17/Q18 reading: hubs scattered over ids)."""
    ks, cs, h, mask = perm_params(seed, s)
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for i in range(3):
            x = x ^ (x >> np.uint64(h))
            x = (x * np.uint64(ks[i]) + np.uint64(cs[i])) & np.uint64(mask)
    return x


RM_T = (2147483648, 2576980377, 3006477107)   # the paper's RM stream: a, b, c = .5, .1, .1


def rmat_pairs(seed: int, s: int, first: int, count: int, permuted: bool = True,
               t=(RMAT_T1, RMAT_T2, RMAT_T3)):
    """RMAT draws first..first+count-1 on 2^s vertices (Graph500 a,b,c = .57,.19,.19
    unless t = floor((a, a+b, a+b+c) * 2^32) says otherwise).

    Level l (0-based, most significant first) uses the 32-bit half (l & 1) of
    mix(seed, RMAT, i*L + l//2), L = ceil(s/2), and sets bit s-1-l of (u, v)."""
    L = (s + 1) // 2
    i = np.arange(first, first + count, dtype=np.uint64)
    u = np.zeros(count, dtype=np.uint64)
    v = np.zeros(count, dtype=np.uint64)
    r = None
    for lvl in range(s):
        if lvl % 2 == 0:
            with np.errstate(over="ignore"):
                r = mix(seed, RMAT_STREAM, i * np.uint64(L) + np.uint64(lvl // 2))
            x = lo32(r)
        else:
            x = hi32(r)
        bit = np.uint64(1) << np.uint64(s - 1 - lvl)
        ub = x >= np.uint64(t[1])                          # quadrants (1,0), (1,1)
        vb = ((x >= np.uint64(t[0])) & (x < np.uint64(t[1]))) | (x >= np.uint64(t[2]))
        u |= np.where(ub, bit, np.uint64(0))
        v |= np.where(vb, bit, np.uint64(0))
    if permuted:
        u = permute(u, seed, s)
        v = permute(v, seed, s)
    return u, v


def csr_from_directed_pairs(n: int, u, v):
    """Symmetrise, drop self-loops, dedup, sort -> (offsets int64[n+1], adj uint32[m])."""
    u = np.asarray(u, dtype=np.uint64)
    v = np.asarray(v, dtype=np.uint64)
    keep = u != v
    u, v = u[keep], v[keep]
    keys = np.concatenate([(u << np.uint64(32)) | v, (v << np.uint64(32)) | u])
    keys = np.unique(keys)
    src = (keys >> np.uint64(32)).astype(np.int64)
    adj = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    off = np.zeros(n + 1, dtype=np.int64)
    if src.size:
        np.cumsum(np.bincount(src, minlength=n), out=off[1:])
    return off, adj


# ---------------------------------------------------------------------------
def er(seed: int = 1, n0: int = 100_000, pairs: int = 400_000, isolated: int = 1_000):
    """C1: `pairs` uniform draws on [0,n0) (u from low, v from high 32 bits of one draw)."""
    r = mix(seed, ER_STREAM, np.arange(pairs, dtype=np.uint64))
    u = scale_u32(lo32(r), n0)
    v = scale_u32(hi32(r), n0)
    return csr_from_directed_pairs(n0 + isolated, u, v)


def grid(seed: int = 2, rows: int = 4096, cols: int = 4096, p32: int = P55):
    """C2: id = r*cols + c; horizontal candidates first, then vertical; keep iff draw < p32."""
    nh = rows * (cols - 1)
    nv = (rows - 1) * cols
    e = np.arange(nh + nv, dtype=np.uint64)
    keep = lo32(mix(seed, GRID_STREAM, e)) < np.uint64(p32)
    eh = e[:nh][keep[:nh]]
    ev = e[nh:][keep[nh:]] - np.uint64(nh)
    rr, cc = eh // np.uint64(cols - 1), eh % np.uint64(cols - 1)
    hu = rr * np.uint64(cols) + cc
    u = np.concatenate([hu, ev])
    v = np.concatenate([hu + np.uint64(1), ev + np.uint64(cols)])
    return csr_from_directed_pairs(rows * cols, u, v)


def rmat(seed: int = 3, scale: int = 24, edge_factor: int = 16, permuted: bool = True):
    """C3/C4: edge_factor * 2^scale RMAT draws, symmetrised/deduplicated/permuted."""
    u, v = rmat_pairs(seed, scale, 0, edge_factor << scale, permuted)
    return csr_from_directed_pairs(1 << scale, u, v)


def incr_batch(seed: int, scale: int, b: int, n_ins: int, n_q: int):
    """C5 batch b: n_ins RMAT-`scale` inserts (draws b*n_ins ..), n_q uniform query pairs.

    Returns (inserts (n_ins,2) uint32, queries (n_q,2) uint32).  Self-loops and
    duplicates are kept (legal no-op inserts, reading R16)."""
    u, v = rmat_pairs(seed, scale, b * n_ins, n_ins, permuted=True)
    n = 1 << scale
    r = mix(seed, QUERY_STREAM, np.arange(b * n_q, (b + 1) * n_q, dtype=np.uint64))
    a = scale_u32(lo32(r), n)
    c = scale_u32(hi32(r), n)
    ins = np.stack([u, v], axis=1).astype(np.uint32)
    qs = np.stack([a, c], axis=1).astype(np.uint32)
    return ins, qs


# ---------------------------------------------------------------------------
# Edge weights for the AMSF workload (NEXT-4): the paper adds "random weights
# drawn from an exponential distribution with a constant mean";
# mean 1 here.  w(u,v) = -ln(U), U = (k + 1/2) 2^-52, k = mix(seed, WEIGHT,
# min(u,v) 2^32 + max(u,v)) >> 12, so both directions of an edge carry the same
# weight and 0 < U < 1 (w > 0).  ln is evaluated with IEEE +,-,*,/ only, in a
# fixed order (no fused multiply-add), so that the CUDA twin (csrc/gen.cu)
# produces bit-identical float32 weights.
LN2 = 0.6931471805599453
LN_TERMS = 10                     # atanh series: t^(2k) / (2k+1), k = 0..LN_TERMS


def _atanh2(t):
    """2 atanh(t) = 2t sum_k t^(2k)/(2k+1) for 0 <= t <= 1/3 (error < 1e-12)."""
    t2 = t * t
    p = np.full_like(t, 1.0 / (2 * LN_TERMS + 1))
    for k in range(LN_TERMS - 1, -1, -1):
        p = p * t2
        p = p + 1.0 / (2 * k + 1)
    return (2.0 * t) * p


def neg_ln_fixed(x) -> np.ndarray:
    """-ln(x) for float64 x in (0, 1).  x < 1/2: x = m 2^e, m in [1, 2),
    -ln x = -(e ln2 + 2 atanh((m-1)/(m+1))); x >= 1/2: d = 1 - x (exact),
    -ln x = 2 atanh(d / (2 - d)) -- no cancellation near x = 1, so the result
    is > 0 for every x < 1."""
    x = np.asarray(x, dtype=np.float64)
    bits = x.view(np.uint64)
    e = ((bits >> np.uint64(52)) & np.uint64(0x7FF)).astype(np.int64) - 1023
    m = ((bits & np.uint64(0x000FFFFFFFFFFFFF)) | np.uint64(1023 << 52)).view(np.float64)
    lo = -(e.astype(np.float64) * LN2 + _atanh2((m - 1.0) / (m + 1.0)))
    d = 1.0 - x
    hi = _atanh2(d / (2.0 - d))
    return np.where(x < 0.5, lo, hi)


def exp_weights(off, adj, seed: int) -> np.ndarray:
    """float32 weight of every adjacency entry (symmetric: w(u,v) == w(v,u))."""
    off = np.asarray(off, dtype=np.int64)
    adj = np.asarray(adj, dtype=np.uint32)
    n = off.size - 1
    src = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off))
    dst = adj.astype(np.uint64)
    key = (np.minimum(src, dst) << np.uint64(32)) | np.maximum(src, dst)
    k = mix(seed, WEIGHT_STREAM, key) >> np.uint64(12)
    u = (k.astype(np.float64) + 0.5) * (2.0 ** -52)
    return neg_ln_fixed(u).astype(np.float32)


def validate_csr(off, adj, n: int | None = None) -> None:
    """Raise AssertionError unless (off, adj) is a valid symmetric sorted simple CSR."""
    off = np.asarray(off, dtype=np.int64)
    adj = np.asarray(adj, dtype=np.uint32)
    n = off.size - 1 if n is None else n
    assert off.size == n + 1 and off[0] == 0 and off[-1] == adj.size
    assert np.all(np.diff(off) >= 0)
    if adj.size == 0:
        return
    assert int(adj.max()) < n
    src = np.repeat(np.arange(n, dtype=np.uint64), np.diff(off))
    keys = (src << np.uint64(32)) | adj.astype(np.uint64)
    assert np.all(np.diff(keys.astype(np.uint64)) > 0), "lists not strictly ascending (dup or unsorted)"
    assert not np.any(src == adj), "self-loop"
    rev = (adj.astype(np.uint64) << np.uint64(32)) | src
    assert np.array_equal(np.sort(rev), keys), "not symmetric"
