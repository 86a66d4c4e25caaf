"""ctypes binding of inputs/libccgen.so: the CUDA twin of inputs/gen.py.

Produces the same bytes as the numpy generator (same seed, same recipe) directly
in device memory, for the full-size configs the numpy generator cannot reach
(RMAT-27: ~4.3e9 directed keys).  Input generation only -- none of the method.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import Config, gen

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libccgen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built (run make)")
        lib = ctypes.CDLL(LIB_PATH)
        U64, P = ctypes.c_uint64, ctypes.c_void_p
        lib.gen_csr_begin.argtypes = [ctypes.c_int, U64, U64, U64, U64, ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_void_p)]
        lib.gen_csr_finish.argtypes = [P, P, P]
        lib.gen_csr_abort.argtypes = [P]
        lib.gen_incr_batch.argtypes = [U64, ctypes.c_int, U64, U64, U64, P, P, P]
        lib.gen_exp_weights.argtypes = [P, P, ctypes.c_uint32, ctypes.c_int64, U64, P, P]
        lib.gen_rmat_stream.argtypes = [U64, ctypes.c_int, U64, U64, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_int, P, P]
        for f in (lib.gen_csr_begin, lib.gen_csr_finish, lib.gen_incr_batch, lib.gen_exp_weights,
                  lib.gen_rmat_stream):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _csr(kind: int, seed: int, p0: int, p1: int, p2: int, device="cuda"):
    lib = _load()
    n = ctypes.c_uint32()
    m = ctypes.c_int64()
    st = ctypes.c_void_p()
    torch.cuda.synchronize()
    rc = lib.gen_csr_begin(kind, seed, p0, p1, p2, ctypes.byref(n), ctypes.byref(m), ctypes.byref(st))
    if rc:
        raise RuntimeError(f"gen_csr_begin failed: {rc}")
    try:
        off = torch.empty(n.value + 1, dtype=torch.int64, device=device)
        adj = torch.empty(max(m.value, 1), dtype=torch.int32, device=device)
    except Exception:
        lib.gen_csr_abort(st)
        raise
    torch.cuda.synchronize()
    rc = lib.gen_csr_finish(st, off.data_ptr(), adj.data_ptr())
    if rc:
        raise RuntimeError(f"gen_csr_finish failed: {rc}")
    return off, adj[:m.value]


def er(seed=1, n0=100_000, pairs=400_000, isolated=1_000):
    return _csr(0, seed, n0, pairs, isolated)


def grid(seed=2, rows=4096, cols=4096, p32=gen.P55):
    return _csr(1, seed, rows, cols, p32)


def rmat(seed=3, scale=24, edge_factor=16, permuted=True):
    return _csr(2, seed, scale, edge_factor, 1 if permuted else 0)


def config_graph(cfg: Config, small: bool = False):
    """Device CSR of a static config (C1-C4)."""
    if cfg.kind == "er":
        return er(cfg.seed)
    if cfg.kind == "grid":
        return grid(cfg.seed, cfg.rows, cfg.cols)
    if cfg.kind == "rmat":
        return rmat(cfg.seed, cfg.scale)
    raise ValueError(cfg.kind)


def incr_batch(seed: int, scale: int, b: int, n_ins: int, n_q: int, ins=None, qs=None, stream=None):
    """Device (inserts (n_ins,2) int32, queries (n_q,2) int32) of stream batch b."""
    ins = torch.empty((n_ins, 2), dtype=torch.int32, device="cuda") if ins is None else ins
    qs = torch.empty((n_q, 2), dtype=torch.int32, device="cuda") if qs is None else qs
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    rc = _load().gen_incr_batch(seed, scale, b, n_ins, n_q, ins.data_ptr(), qs.data_ptr(), s)
    if rc:
        raise RuntimeError(f"gen_incr_batch failed: {rc}")
    return ins, qs


def exp_weights(d_off, d_adj, seed: int, stream=None):
    """Device float32 weights aligned with d_adj (gen.exp_weights' bytes)."""
    n, m = d_off.numel() - 1, d_adj.numel()
    w = torch.empty(max(m, 1), dtype=torch.float32, device=d_adj.device)
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    rc = _load().gen_exp_weights(d_off.data_ptr(), d_adj.data_ptr(), n, m, seed, w.data_ptr(), s)
    if rc:
        raise RuntimeError(f"gen_exp_weights failed: {rc}")
    return w[:m]


def rmat_stream(seed: int, s: int, first: int, count: int, t=gen.RM_T, permuted: bool = False, out=None,
                stream=None):
    """Device (count, 2) int32 RMAT pairs (gen.rmat_pairs' values) -- the Table 4 RM stream by default."""
    out = torch.empty((count, 2), dtype=torch.int32, device="cuda") if out is None else out
    st = torch.cuda.current_stream().cuda_stream if stream is None else stream
    rc = _load().gen_rmat_stream(seed, s, first, count, t[0], t[1], t[2], 1 if permuted else 0, out.data_ptr(), st)
    if rc:
        raise RuntimeError(f"gen_rmat_stream failed: {rc}")
    return out
