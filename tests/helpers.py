"""Shared test helpers: fixture graphs (hand-built CSRs) and device transfer."""
from __future__ import annotations

import os

import numpy as np


def csr(n, pairs, keep_dups=False, keep_loops=False):
    """Symmetric CSR with sorted lists; optionally keep duplicate entries / self-loops."""
    lists = [[] for _ in range(n)]
    for u, v in pairs:
        if u == v:
            if keep_loops:
                lists[u].append(v)
            continue
        lists[u].append(v)
        lists[v].append(u)
    off = np.zeros(n + 1, dtype=np.int64)
    flat = []
    for i in range(n):
        li = sorted(lists[i]) if keep_dups else sorted(set(lists[i]))
        flat += li
        off[i + 1] = off[i] + len(li)
    return off, np.array(flat, dtype=np.uint32)


def fixtures():
    """(name, off, adj) covering the edge cases of SURVEY §8(c)."""
    F = []
    F.append(("n1", *csr(1, [])))
    F.append(("edgeless9", *csr(9, [])))
    F.append(("one_edge", *csr(2, [(0, 1)])))
    F.append(("one_edge_far", *csr(7, [(6, 2)])))
    F.append(("counter_example", *csr(6, [(0, 2), (1, 3), (2, 5), (3, 4), (4, 5)])))
    n = 64
    F.append(("star_center_last", *csr(n, [(n - 1, i) for i in range(n - 1)])))
    F.append(("star_center_first", *csr(n, [(0, i) for i in range(1, n)])))
    F.append(("path_decreasing", *csr(300, [(i + 1, i) for i in range(299)])))
    F.append(("path_zigzag", *csr(200, [(i, 199 - i) for i in range(100)] + [(199 - i, i + 1) for i in range(99)])))
    F.append(("deg0_ends", *csr(12, [(1, 2), (2, 3), (5, 9), (9, 10)])))
    # two equal-size giants (L_max tie), plus small pieces
    a = [(i, i + 1) for i in range(0, 49)]
    b = [(i, i + 1) for i in range(50, 99)]
    F.append(("two_giants", *csr(110, a + b + [(100, 101), (105, 106)])))
    # the sampled L_max component later merges with a smaller-id component:
    # star 1 -- {10..209} is the sampled giant (root 1); path 0-2-3 has root 0;
    # the join (3, 100) is the second entry of both lists, so with k = 1 it is
    # applied only in the finish, which hooks root 1 under 0 and H6 must
    # relabel the whole giant
    big = [(1, i) for i in range(10, 210)]
    F.append(("lmax_merges_smaller", *csr(210, big + [(0, 2), (2, 3), (3, 100)])))
    F.append(("cliques", *csr(7 * 5, [(b * 5 + i, b * 5 + j) for b in range(7) for i in range(5) for j in range(i + 1, 5)])))
    F.append(("dups_and_loops", *csr(8, [(0, 1), (0, 1), (1, 2), (3, 3), (4, 5), (5, 4), (6, 6)],
                                     keep_dups=True, keep_loops=True)))
    R, C = 23, 31
    g = [(r * C + c, r * C + c + 1) for r in range(R) for c in range(C - 1)]
    g += [(r * C + c, (r + 1) * C + c) for r in range(R - 1) for c in range(C)]
    F.append(("full_grid", *csr(R * C, g)))
    # hub with a list longer than the CTA threshold (4096) and a medium hub
    hub = [(0, i) for i in range(1, 6001)] + [(6001, i) for i in range(6002, 6300)]
    F.append(("hubs", *csr(6400, hub)))
    return F


def to_dev(off, adj, device="cuda"):
    import torch
    d_off = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).to(device)
    d_adj = torch.from_numpy(np.ascontiguousarray(adj, dtype=np.uint32).view(np.int32)).to(device)
    return d_off, d_adj


def u32(t):
    return t.detach().cpu().numpy().view(np.uint32)


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_fixtures():
    """tests/golden/*.txt: small graphs with paper-cited expected values.
    Yields (name, off, adj, expect) with expect = {components, labels, forest_edges}."""
    for fn in sorted(os.listdir(GOLDEN)):
        if not fn.endswith(".txt"):
            continue
        kv = {}
        for line in open(os.path.join(GOLDEN, fn)):
            line = line.split("#", 1)[0].strip()
            if line:
                k, *vals = line.split()
                kv[k] = [int(x) for x in vals]
        n = kv["n"][0]
        e = kv["edges"]
        pairs = list(zip(e[0::2], e[1::2]))
        off, adj = csr(n, pairs)
        yield fn, off, adj, {"components": kv["components"][0], "labels": np.array(kv["labels"], dtype=np.uint32),
                             "forest_edges": kv["forest_edges"][0]}
