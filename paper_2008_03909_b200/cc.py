"""Thin ctypes binding of libcc.so (include/cc.h, include/cc_bench.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of ``csrc/``.  Tensors supply device (or host) pointers via
``data_ptr()`` and the current torch stream supplies ``cudaStream_t``.  There
is no CPU fallback: if libcc.so is missing or fails to load, every call raises.

Dtypes: PyTorch's uint32 has limited op support, so ids/labels are passed as
``torch.int32`` tensors and reinterpreted as uint32 by the C side
(``labels.cpu().numpy().view(np.uint32)`` on the host); offsets are
``torch.int64``; answers ``torch.uint8``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CC_LIBCC_PATH overrides the library (A/B measurements of build variants only)
LIB_PATH = os.environ.get("CC_LIBCC_PATH") or os.path.join(_HERE, "libcc.so")

CC_OK, CC_EINVAL, CC_ERANGE, CC_ENOMEM, CC_ECUDA = 0, -1, -2, -3, -4
VARIANT_AFFOREST, VARIANT_HYBRID, VARIANT_PURE = 0, 1, 2
FLAG_NO_SKIP = 1 << 0
FLAG_VALIDATE = 1 << 1
FLAG_UF_ASYNC = 1 << 2
FLAG_HALVE = 1 << 3
FLAG_FIND_SPLIT = 1 << 4
FLAG_NO_DEGSKIP = 1 << 5
FLAG_NO_MIDCOMPRESS = 1 << 6
FLAG_MIDCOMPRESS = 1 << 7
FLAG_WAIT_FREE = 1 << 8
FLAG_FINISH_SV = 1 << 9
FLAG_CONTRACT = 1 << 10
FLAG_NO_REFILL = 1 << 11
FLAG_AMSF_PLAIN = 1 << 12
FLAG_FINISH_CRFA = 1 << 13
FLAG_AMSF_NO_INDEX = 1 << 14
FLAG_FUSED_LINK = 1 << 16
FLAG_FIND_NAIVE = 1 << 15
FLAG_LINK_REFILL = 1 << 18

# every symbol include/cc.h and include/cc_bench.h declare
EXPORTS = [
    "cc_opts_default", "cc_labels", "cc_spanning_forest", "cc_incr_create", "cc_incr_batch",
    "cc_incr_batches", "cc_incr_labels", "cc_incr_destroy", "cc_incr_num_vertices", "cc_status_str", "cc_last_error",
    "cc_amsf",
    "cc_workspace_bytes", "cc_version",
    "cc_bench_map_edges", "cc_bench_gather_edges", "cc_bench_random_gather", "cc_bench_copy",
    "cc_bench_launch_count", "cc_bench_set_l2_fetch", "cc_bench_set_grid",
]


class Timings(ctypes.Structure):
    _fields_ = [("sample_ms", ctypes.c_float), ("identify_ms", ctypes.c_float), ("finish_ms", ctypes.c_float),
                ("compress_ms", ctypes.c_float), ("total_ms", ctypes.c_float)]

    def as_dict(self):
        return {f: float(getattr(self, f)) for f, _ in self._fields_}


COUNTER_FIELDS = ["pending_links", "worklist", "finish_vertices", "finish_edges", "sample_hooks", "finish_hooks",
                  "big_vertices", "compress_writes",
                  "link_steps", "cas_failures", "probe_deep", "finish_gathers", "h6_writes", "h6_gathers",
                  "sv_rounds", "contract_roots", "amsf_rounds", "amsf_visits", "amsf_edges", "amsf_hooks",
                  "amsf_rebuilds", "fused_link", "amsf_links", "h6_tiles", "link_pending", "mid_compress"]


class Opts(ctypes.Structure):
    _fields_ = [("kout_k", ctypes.c_uint32), ("kout_variant", ctypes.c_uint32), ("seed", ctypes.c_uint64),
                ("samples", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("sampled_out", ctypes.c_void_p), ("lmax_out", ctypes.c_void_p), ("lmax_force", ctypes.c_void_p),
                ("counters", ctypes.c_void_p), ("timings", ctypes.POINTER(Timings)),
                ("marks", ctypes.POINTER(ctypes.c_void_p))]


NUM_MARKS = 10
MARK_NAMES = ["start", "k_sample_init", "k_compress_mid", "k_link_pending", "k_compress_H3_debug", "k_identify",
              "k_finish", "k_finish_proc", "k_compress_H6", "k_forest"]


class CCError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    """Load libcc.so (raises loudly if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CCError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    P, U32, I64, U64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int64, ctypes.c_uint64
    OP = ctypes.POINTER(Opts)
    sig = {
        "cc_opts_default": (None, [OP]),
        "cc_labels": (ctypes.c_int, [P, P, U32, I64, P, OP, P]),
        "cc_spanning_forest": (ctypes.c_int, [P, P, U32, I64, P, P, P, OP, P]),
        "cc_amsf": (ctypes.c_int, [P, P, P, U32, I64, ctypes.c_double, P, P, P, P, OP, P]),
        "cc_incr_create": (ctypes.c_int, [U32, OP, P, ctypes.POINTER(ctypes.c_void_p)]),
        "cc_incr_batch": (ctypes.c_int, [P, P, I64, P, I64, P, P]),
        "cc_incr_batches": (ctypes.c_int, [P, I64, P, P, P, P, P, P]),
        "cc_incr_labels": (ctypes.c_int, [P, P, P]),
        "cc_incr_destroy": (None, [P]),
        "cc_incr_num_vertices": (U32, [P]),
        "cc_status_str": (ctypes.c_char_p, [ctypes.c_int]),
        "cc_last_error": (ctypes.c_char_p, []),
        "cc_workspace_bytes": (ctypes.c_size_t, [U32, I64, U32, ctypes.c_int]),
        "cc_version": (ctypes.c_char_p, []),
        "cc_bench_map_edges": (ctypes.c_int, [P, P, U32, P, P]),
        "cc_bench_gather_edges": (ctypes.c_int, [P, P, U32, P, P, P]),
        "cc_bench_random_gather": (ctypes.c_int, [P, U64, U64, U64, P, P]),
        "cc_bench_copy": (ctypes.c_int, [P, P, U64, P]),
        "cc_bench_launch_count": (U64, []),
        "cc_bench_set_l2_fetch": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "cc_bench_set_grid": (ctypes.c_uint, [ctypes.c_uint]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("CC_LIBCC_PATH") and not hasattr(lib, name):
            continue                    # an older A/B build may lack a newer bench-only symbol
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != CC_OK:
        lib = load()
        raise CCError(f"{what}: {lib.cc_status_str(rc).decode()} ({lib.cc_last_error().decode()})", rc)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data           # numpy (host buffer)


def _stream(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream().cuda_stream
        return None
    return stream if isinstance(stream, int) else stream.cuda_stream


def make_opts(k=2, variant=VARIANT_AFFOREST, seed=0, samples=1024, flags=0, sampled_out=None, lmax_out=None,
              lmax_force=None, counters=None, timings: Timings | None = None, marks=None) -> Opts:
    o = Opts()
    o.kout_k, o.kout_variant, o.seed, o.samples, o.flags = k, variant, seed, samples, flags
    o.sampled_out, o.lmax_out, o.lmax_force = _ptr(sampled_out), _ptr(lmax_out), _ptr(lmax_force)
    o.counters = _ptr(counters)
    o.timings = ctypes.pointer(timings) if timings is not None else None
    if marks is not None:        # list of NUM_MARKS raw cudaEvent_t handles
        arr = (ctypes.c_void_p * NUM_MARKS)(*marks)
        o._marks_keepalive = arr
        o.marks = ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))
    return o


def cc_labels(offsets, adj, n, m, labels, opts: Opts | None = None, stream=None):
    """Canonical connectivity labels into `labels` (int32/uint32 tensor of n)."""
    rc = load().cc_labels(_ptr(offsets), _ptr(adj), n, m, _ptr(labels),
                          ctypes.byref(opts) if opts is not None else None, _stream(stream))
    _check(rc, "cc_labels")


def cc_spanning_forest(offsets, adj, n, m, edges, num_edges, labels=None, opts: Opts | None = None, stream=None):
    rc = load().cc_spanning_forest(_ptr(offsets), _ptr(adj), n, m, _ptr(edges), _ptr(num_edges), _ptr(labels),
                                   ctypes.byref(opts) if opts is not None else None, _stream(stream))
    _check(rc, "cc_spanning_forest")


def cc_amsf(offsets, adj, w, n, m, eps, edges, edge_w, num_edges, total=None, opts: Opts | None = None,
            stream=None):
    """AMSF-NF-S (include/cc.h cc_amsf); every array is a device tensor."""
    rc = load().cc_amsf(_ptr(offsets), _ptr(adj), _ptr(w), n, m, float(eps), _ptr(edges), _ptr(edge_w),
                        _ptr(num_edges), _ptr(total), ctypes.byref(opts) if opts is not None else None,
                        _stream(stream))
    _check(rc, "cc_amsf")


class Incr:
    """Handle over cc_incr_create / cc_incr_batch / cc_incr_labels / cc_incr_destroy."""

    def __init__(self, n: int, flags: int = 0, stream=None):
        self._lib = load()
        h = ctypes.c_void_p()
        o = make_opts(flags=flags)
        _check(self._lib.cc_incr_create(n, ctypes.byref(o), _stream(stream), ctypes.byref(h)), "cc_incr_create")
        self.h = h
        self.n = n

    def batch(self, inserts, n_ins, queries, n_q, answers, stream=None):
        _check(self._lib.cc_incr_batch(self.h, _ptr(inserts), n_ins, _ptr(queries), n_q, _ptr(answers),
                                       _stream(stream)), "cc_incr_batch")

    def batches(self, ins_counts, inserts, q_counts, queries, answers, stream=None):
        """nb batches in one call; counts are int64 numpy arrays (host)."""
        import numpy as np
        ic = np.ascontiguousarray(ins_counts, dtype=np.int64)
        qc = np.ascontiguousarray(q_counts, dtype=np.int64)
        _check(self._lib.cc_incr_batches(self.h, ic.size, ic.ctypes.data, _ptr(inserts), qc.ctypes.data,
                                         _ptr(queries), _ptr(answers), _stream(stream)), "cc_incr_batches")

    def labels(self, out, stream=None):
        _check(self._lib.cc_incr_labels(self.h, _ptr(out), _stream(stream)), "cc_incr_labels")

    def close(self):
        if self.h:
            self._lib.cc_incr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def map_edges(offsets, adj, n, out, stream=None):
    _check(load().cc_bench_map_edges(_ptr(offsets), _ptr(adj), n, _ptr(out), _stream(stream)), "map_edges")


def gather_edges(offsets, adj, n, x, out, stream=None):
    _check(load().cc_bench_gather_edges(_ptr(offsets), _ptr(adj), n, _ptr(x), _ptr(out), _stream(stream)),
           "gather_edges")


def random_gather(x, length, count, seed, out, stream=None):
    _check(load().cc_bench_random_gather(_ptr(x), length, count, seed, _ptr(out), _stream(stream)), "random_gather")


def copy(src, dst, words, stream=None):
    _check(load().cc_bench_copy(_ptr(src), _ptr(dst), words, _stream(stream)), "copy")


def set_l2_fetch(nbytes: int) -> int:
    prev = ctypes.c_int()
    _check(load().cc_bench_set_l2_fetch(nbytes, ctypes.byref(prev)), "set_l2_fetch")
    return prev.value


def set_grid(blocks: int) -> int:
    """Test hook: grid-strided kernels launch exactly `blocks` blocks (0 = default)."""
    return int(load().cc_bench_set_grid(blocks))


def launch_count() -> int:
    return int(load().cc_bench_launch_count())
