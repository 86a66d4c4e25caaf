"""oracle -- TEST INFRASTRUCTURE ONLY (arXiv 2008.03909, ConnectIt).

The plain, slow, obviously-correct CPU oracle of the connectivity hot path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA product (``paper_2008_03909_b200``) and neither
imports the other; the only common dependency is ``inputs`` (seeded input
generators, none of the method's arithmetic).

Contents (each cites the PAPER.md passage it follows):

* ``cc_bfs`` / ``cc_dsu`` -- canonical connectivity labels (min-id
  canonical form per the north_star, reading R13), from ``oracle.c``.
* ``forest_check`` -- spanning-forest validity triple (Alg. 2
  P:2406-2418).
* ``incr_run`` -- batch-incremental answers (inserts of
  a batch are visible to its queries, reading R15 / P:986-993).
* ``kout_sample_edges`` -- the edge set k-out sampling unions (Alg. 4
  P:3947-3958; afforest "first k" P:3589-3591; hybrid "first + k-1 uniform"
  P:616-619), so that the sampled partition (height-one labels after the
  sampling compress, Def. 3.1) is ``cc_bfs`` of that edge set.
* ``identify_frequent`` -- IdentifyFrequent (Alg. 1 line 5):
  the most frequent label among S seeded samples, ties to the smaller label
  (reading R9).
* ``canon`` -- map every label class to its minimum member (reading R13).
* ``kruskal`` -- exact minimum spanning forest W(F_OPT), from
  ``oracle.c``.
* ``amsf`` -- the folklore AMSF algorithm step by step: W_min,
  (1+eps)-buckets (reading R25), per-bucket spanning forests over the
  labeling, from ``oracle.c``; ``amsf_bounds`` / ``amsf_bucket`` restate the
  bucket rule in numpy (same fp64 product chain) for checking a forest.

Random draws the method makes (hybrid picks, IdentifyFrequent samples) use the
counter-based generator of reading R7/R9, re-implemented here independently of
the CUDA side: ``mix(seed, stream, i) = splitmix64(seed*GOLD + stream*2^40 + i)``.

Parity status: every function above is pinned in ``tests/test_oracle.py``
(brute force, closed forms, scipy, cross-oracle agreement) except
``kout_sample_edges`` / ``identify_frequent``, whose *choice* of edges/samples
is a reading of the paper (R7, R9) pinned only by closed-form special cases.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (building the checker is not using it)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", src, "-o", _LIB_PATH])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.oracle_cc_bfs.argtypes = [ctypes.c_uint32, P, P, P]
        lib.oracle_cc_dsu.argtypes = [ctypes.c_uint32, P, P, P]
        lib.oracle_forest_check.argtypes = [ctypes.c_uint32, P, P, ctypes.c_uint64, P, ctypes.c_int64,
                                            ctypes.POINTER(ctypes.c_int64)]
        lib.oracle_incr_run.argtypes = [ctypes.c_uint32, ctypes.c_int64, P, P, P, P, P, P]
        D, I64P = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        lib.oracle_kruskal.argtypes = [ctypes.c_uint32, P, P, P, D, P, P, I64P]
        lib.oracle_amsf.argtypes = [ctypes.c_uint32, P, P, P, ctypes.c_double, D, P, P, P, I64P, I64P]
        for f in (lib.oracle_cc_bfs, lib.oracle_cc_dsu, lib.oracle_forest_check, lib.oracle_incr_run,
                  lib.oracle_kruskal, lib.oracle_amsf):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _csr(off, adj):
    off = np.ascontiguousarray(off, dtype=np.int64)
    adj = np.ascontiguousarray(adj, dtype=np.uint32)
    if adj.size == 0:
        adj = np.zeros(1, dtype=np.uint32)     # valid pointer for m = 0
    return off, adj


def cc_bfs(off, adj) -> np.ndarray:
    """lab[v] = min vertex id of v's component, by BFS in id order."""
    off, adj = _csr(off, adj)
    n = off.size - 1
    lab = np.empty(max(n, 1), dtype=np.uint32)
    rc = _load().oracle_cc_bfs(n, _ptr(off), _ptr(adj), _ptr(lab))
    if rc:
        raise ValueError(f"oracle_cc_bfs failed: {rc}")
    return lab[:n]


def cc_dsu(off, adj) -> np.ndarray:
    """Same labels via a sequential union-find, then min per set."""
    off, adj = _csr(off, adj)
    n = off.size - 1
    lab = np.empty(max(n, 1), dtype=np.uint32)
    rc = _load().oracle_cc_dsu(n, _ptr(off), _ptr(adj), _ptr(lab))
    if rc:
        raise ValueError(f"oracle_cc_dsu failed: {rc}")
    return lab[:n]


FOREST_ERRORS = {0: "ok", 1: "count != n - c", 2: "endpoint out of range", 3: "self-loop pair",
                 4: "pair is not an input edge", 5: "pair closes a cycle"}


def forest_check(off, adj, num_components: int, F) -> tuple[int, int]:
    """(code, bad_index) for a candidate spanning forest F (pairs). 0 = valid."""
    off, adj = _csr(off, adj)
    n = off.size - 1
    F = np.ascontiguousarray(np.asarray(F, dtype=np.uint32).reshape(-1))
    nf = F.size // 2
    Fb = F if F.size else np.zeros(2, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_forest_check(n, _ptr(off), _ptr(adj), int(num_components), _ptr(Fb), nf,
                                     ctypes.byref(bad))
    if rc < 0:
        raise MemoryError("oracle_forest_check")
    return rc, bad.value


def incr_run(n: int, batches, want_labels: bool = False):
    """Sequential union-find over batches [(inserts (k,2), queries (q,2)), ...].

    Returns (answers uint8 concatenated over batches, final labels or None).
    A query sees all inserts of batches 0..b inclusive (reading R15)."""
    nb = len(batches)
    ins_cnt = np.array([np.asarray(b[0]).reshape(-1, 2).shape[0] for b in batches] or [0], dtype=np.int64)
    q_cnt = np.array([np.asarray(b[1]).reshape(-1, 2).shape[0] for b in batches] or [0], dtype=np.int64)
    ins = np.concatenate([np.asarray(b[0], dtype=np.uint32).reshape(-1) for b in batches] + [np.zeros(2, np.uint32)])
    qs = np.concatenate([np.asarray(b[1], dtype=np.uint32).reshape(-1) for b in batches] + [np.zeros(2, np.uint32)])
    ans = np.zeros(int(q_cnt[:nb].sum()) + 1, dtype=np.uint8)
    lab = np.empty(max(n, 1), dtype=np.uint32) if want_labels else None
    rc = _load().oracle_incr_run(n, nb, _ptr(ins_cnt), _ptr(np.ascontiguousarray(ins)), _ptr(q_cnt),
                                 _ptr(np.ascontiguousarray(qs)), _ptr(ans),
                                 _ptr(lab) if want_labels else None)
    if rc:
        raise ValueError(f"oracle_incr_run failed: {rc}")
    return ans[:-1], (lab[:n] if want_labels else None)


# ---------------------------------------------------------------------------
# Plain statements of the method's choices (sampling edge set, L_max samples).
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15
KOUT_STREAM = 16       # hybrid random picks:   index = u * 64 + j
IDENT_STREAM = 17      # IdentifyFrequent draws: index = i


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(GOLD)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def mix(seed: int, stream: int, idx) -> np.ndarray:
    base = np.uint64(((seed * GOLD) + (stream << 40)) & _M64)
    with np.errstate(over="ignore"):
        return splitmix64(np.asarray(idx, dtype=np.uint64) + base)


def uniform_below(r: np.ndarray, bound) -> np.ndarray:
    """Multiply-shift map of the low 32 bits of r onto [0, bound)."""
    lo = r & np.uint64(0xFFFFFFFF)
    return ((lo * np.asarray(bound, dtype=np.uint64)) >> np.uint64(32)).astype(np.uint64)


def kout_sample_edges(off, adj, k: int, variant: str = "afforest", seed: int = 0) -> np.ndarray:
    """The edge set k-out sampling unions (Alg. 4).

    afforest: adjacency positions 0..min(k,deg)-1 ("first k").
    hybrid:   position 0, then k-1 positions drawn uniformly with replacement
              (P:616-619), i = uniform_below(mix(seed, KOUT, u*64+j), deg).
    pure:     k positions drawn that way, j = 0..k-1 (Holm et al.).
    Returns an (E, 2) uint32 array of (u, v) pairs."""
    off = np.asarray(off, dtype=np.int64)
    adj = np.asarray(adj, dtype=np.uint32)
    n = off.size - 1
    deg = np.diff(off)
    us, vs = [], []
    for j in range(k):
        has = deg > j if variant == "afforest" else deg > 0
        u = np.nonzero(has)[0].astype(np.uint64)
        if u.size == 0:
            continue
        if variant == "afforest" or (variant == "hybrid" and j == 0):
            pos = off[u.astype(np.int64)] + j
        elif variant in ("hybrid", "pure"):
            r = mix(seed, KOUT_STREAM, u * np.uint64(64) + np.uint64(j))
            pos = off[u.astype(np.int64)] + uniform_below(r, deg[u.astype(np.int64)].astype(np.uint64)).astype(np.int64)
        else:
            raise ValueError(variant)
        us.append(u.astype(np.uint32))
        vs.append(adj[pos])
    if not us:
        return np.zeros((0, 2), dtype=np.uint32)
    del n
    return np.stack([np.concatenate(us), np.concatenate(vs)], axis=1)


def csr_from_pairs(n: int, pairs) -> tuple[np.ndarray, np.ndarray]:
    """Symmetric CSR (sorted, deduplicated) of an undirected pair list."""
    pairs = np.asarray(pairs, dtype=np.uint64).reshape(-1, 2)
    u = np.concatenate([pairs[:, 0], pairs[:, 1]])
    v = np.concatenate([pairs[:, 1], pairs[:, 0]])
    keys = np.unique((u << np.uint64(32)) | v)
    src = (keys >> np.uint64(32)).astype(np.int64)
    adj = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=off[1:])
    return off, adj


def sample_positions(n: int, samples: int, seed: int) -> np.ndarray:
    """IdentifyFrequent sample vertices s_i = uniform_below(mix(seed, IDENT, i), n)."""
    return uniform_below(mix(seed, IDENT_STREAM, np.arange(samples, dtype=np.uint64)), n).astype(np.int64)


def identify_frequent(sampled_labels: np.ndarray, samples: int, seed: int) -> int:
    """Mode of the labels at the sample positions; ties -> smaller label (R9)."""
    n = sampled_labels.size
    vals = np.asarray(sampled_labels)[sample_positions(n, samples, seed)]
    uniq, cnt = np.unique(vals, return_counts=True)   # uniq ascending => argmax picks smallest tie
    return int(uniq[int(np.argmax(cnt))])


def canon(labels) -> np.ndarray:
    """Map each label class to its minimum member id (reading R13)."""
    labels = np.asarray(labels, dtype=np.int64)
    n = labels.size
    if n == 0:
        return labels.astype(np.uint32)
    mn = np.full(int(labels.max()) + 1, np.iinfo(np.int64).max, dtype=np.int64)
    np.minimum.at(mn, labels, np.arange(n, dtype=np.int64))
    return mn[labels].astype(np.uint32)


# ---------------------------------------------------------------------------
# Minimum spanning forests: exact (Kruskal) and the AMSF folklore algorithm.
# ---------------------------------------------------------------------------
def _weights(off, w):
    w = np.ascontiguousarray(w, dtype=np.float32)
    if w.size == 0:
        w = np.zeros(1, dtype=np.float32)
    return w


def kruskal(off, adj, w):
    """Exact MSF: (total weight fp64, pairs (k,2) uint32, weights (k,) f32)."""
    off, adj = _csr(off, adj)
    n = off.size - 1
    w = _weights(off, w)
    F = np.zeros(2 * max(n, 1), dtype=np.uint32)
    Fw = np.zeros(max(n, 1), dtype=np.float32)
    tot = ctypes.c_double()
    nf = ctypes.c_int64()
    rc = _load().oracle_kruskal(n, _ptr(off), _ptr(adj), _ptr(w), ctypes.byref(tot), _ptr(F), _ptr(Fw),
                                ctypes.byref(nf))
    if rc:
        raise ValueError(f"oracle_kruskal failed: {rc}")
    k = nf.value
    return tot.value, F[:2 * k].reshape(-1, 2), Fw[:k]


def amsf(off, adj, w, eps: float):
    """AMSF folklore algorithm.  Returns a dict with the forest
    pairs, their weights and bucket indices (in the order added), the fp64
    total and the bucket count."""
    off, adj = _csr(off, adj)
    n = off.size - 1
    w = _weights(off, w)
    F = np.zeros(2 * max(n, 1), dtype=np.uint32)
    Fw = np.zeros(max(n, 1), dtype=np.float32)
    Fb = np.zeros(max(n, 1), dtype=np.int32)
    tot = ctypes.c_double()
    nf = ctypes.c_int64()
    nb = ctypes.c_int64()
    rc = _load().oracle_amsf(n, _ptr(off), _ptr(adj), _ptr(w), float(eps), ctypes.byref(tot), _ptr(F), _ptr(Fw),
                             _ptr(Fb), ctypes.byref(nf), ctypes.byref(nb))
    if rc:
        raise ValueError(f"oracle_amsf failed: {rc}")
    k = nf.value
    return {"total": tot.value, "pairs": F[:2 * k].reshape(-1, 2), "weights": Fw[:k], "buckets": Fb[:k],
            "nbuckets": nb.value}


def amsf_bounds(wmin: float, wmax: float, eps: float) -> np.ndarray:
    """Bucket boundaries b_0 = W_min, b_(i+1) = b_i (1+eps) in fp64 (reading R25),
    up to the first one above W_max."""
    g = 1.0 + float(eps)
    b = [float(np.float32(wmin))]
    while b[-1] * g <= float(np.float32(wmax)):
        b.append(b[-1] * g)
    b.append(b[-1] * g)
    return np.array(b, dtype=np.float64)


def amsf_bucket(w, bounds: np.ndarray) -> np.ndarray:
    """Bucket index i with b_i <= w < b_(i+1) of float32 weights w."""
    return (np.searchsorted(bounds, np.asarray(w, dtype=np.float32).astype(np.float64), side="right") - 1).astype(np.int64)
