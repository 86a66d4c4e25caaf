"""paper_2008_03909_b200 -- ConnectIt's connectivity hot path on one B200.

Public API (torch tensors in, torch tensors out; all compute in libcc.so):

* ``connected_components(offsets, adj, k=2, variant="afforest", ...)`` ->
  int32 labels (canonical: min vertex id of each component).
* ``spanning_forest(offsets, adj, ...)`` -> (edges (F,2) int32, labels).
* ``amsf(offsets, adj, w, eps=0.25)`` -> (edges (F,2) int32, weights (F,) f32,
  total weight): an approximate minimum spanning forest (AMSF-NF-S).
* ``IncrementalCC(n)`` with ``.batch(inserts, queries)`` -> uint8 answers and
  ``.labels()``.

The C ABI is ``include/cc.h``; ``cc`` is the ctypes binding of it.
"""
from __future__ import annotations

from . import cc
from .cc import CCError  # noqa: F401

_VARIANTS = {"afforest": cc.VARIANT_AFFOREST, "hybrid": cc.VARIANT_HYBRID, "pure": cc.VARIANT_PURE}


def _opts(k, variant, seed, flags, **kw):
    return cc.make_opts(k=k, variant=_VARIANTS[variant], seed=seed, flags=flags, **kw)


def connected_components(offsets, adj, k: int = 2, variant: str = "afforest", seed: int = 0, flags: int = 0,
                         out=None, stream=None, **hooks):
    """Canonical CC labels of the symmetric CSR (offsets int64[n+1], adj int32/uint32[m])."""
    import torch
    n = offsets.numel() - 1
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int32, device=offsets.device)
    cc.cc_labels(offsets, adj, n, adj.numel(), out, _opts(k, variant, seed, flags, **hooks), stream)
    return out


def spanning_forest(offsets, adj, k: int = 2, variant: str = "afforest", seed: int = 0, flags: int = 0,
                    with_labels: bool = True, stream=None, **hooks):
    """A spanning forest (pairs (u, v), v in N(u)) and, optionally, the canonical labels."""
    import torch
    n = offsets.numel() - 1
    dev = offsets.device
    edges = torch.empty((max(n, 1), 2), dtype=torch.int32, device=dev)
    num = torch.zeros(1, dtype=torch.int64, device=dev)
    labels = torch.empty(max(n, 0), dtype=torch.int32, device=dev) if with_labels else None
    cc.cc_spanning_forest(offsets, adj, n, adj.numel(), edges, num, labels, _opts(k, variant, seed, flags, **hooks),
                          stream)
    ne = int(num.item())
    return edges[:ne], labels


def amsf(offsets, adj, w, eps: float = 0.25, flags: int = 0, seed: int = 0, samples: int = 1024, stream=None,
         **hooks):
    """AMSF-NF-S (Sec. 5.1): W(F_OPT) <= W(F) <= (1+eps) W(F_OPT) for symmetric
    positive float32 weights w aligned with adj."""
    import torch
    n = offsets.numel() - 1
    dev = offsets.device
    edges = torch.empty((max(n, 1), 2), dtype=torch.int32, device=dev)
    ew = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    num = torch.zeros(1, dtype=torch.int64, device=dev)
    tot = torch.zeros(1, dtype=torch.float64, device=dev)
    cc.cc_amsf(offsets, adj, w, n, adj.numel(), eps, edges, ew, num, tot,
               cc.make_opts(seed=seed, samples=samples, flags=flags, **hooks), stream)
    ne = int(num.item())
    return edges[:ne], ew[:ne], float(tot.item())


class IncrementalCC:
    """Batch-incremental connectivity over a persistent parent array (Alg. 3)."""

    def __init__(self, n: int, flags: int = 0, stream=None):
        self._h = cc.Incr(n, flags, stream)
        self.n = n

    def batch(self, inserts, queries, answers=None, stream=None):
        import torch
        nq = queries.shape[0] if queries is not None else 0
        if answers is None:
            answers = torch.empty(nq, dtype=torch.uint8, device=queries.device if nq else "cuda")
        self._h.batch(inserts, inserts.shape[0] if inserts is not None else 0, queries, nq, answers, stream)
        return answers

    def labels(self, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.n, dtype=torch.int32, device="cuda")
        self._h.labels(out, stream)
        return out

    def close(self):
        self._h.close()
