"""CPU-side checks of the C ABI: libcc.so loads, exports every symbol include/*.h
declares, and the host-side argument checks answer without touching a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2008_03909_b200 import cc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in ("cc.h", "cc_bench.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cc_\w+)\s*\(", src, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_all_declared_symbols_exported():
    lib = cc.load()
    syms = declared_symbols()
    assert len(syms) >= 17
    assert syms == set(cc.EXPORTS), syms ^ set(cc.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_no_oracle_linkage():
    # the product library must not link or name the oracle
    data = open(cc.LIB_PATH, "rb").read()
    assert b"oracle" not in data
    assert b"liboracle" not in data


def test_host_argument_checks_no_gpu():
    lib = cc.load()
    o = cc.Opts()
    lib.cc_opts_default(ctypes.byref(o))
    assert (o.kout_k, o.kout_variant, o.samples, o.flags) == (2, 0, 1024, 0)
    assert lib.cc_status_str(cc.CC_EINVAL) == b"CC_EINVAL"
    # n too large -> CC_ERANGE before any CUDA call
    assert lib.cc_labels(None, None, 0xFFFFFFFF, 0, None, None, None) == cc.CC_ERANGE
    # negative m, null offsets
    assert lib.cc_labels(None, None, 10, -1, None, None, None) == cc.CC_EINVAL
    assert lib.cc_labels(None, None, 10, 0, None, None, None) == cc.CC_EINVAL
    bad = cc.make_opts(k=65)
    off = np.zeros(11, np.int64)
    assert lib.cc_labels(off.ctypes.data, None, 10, 0, off.ctypes.data, ctypes.byref(bad), None) == cc.CC_ERANGE
    bad = cc.make_opts(variant=7)
    assert lib.cc_labels(off.ctypes.data, None, 10, 0, off.ctypes.data, ctypes.byref(bad), None) == cc.CC_EINVAL
    # n = 0 is a no-op
    assert lib.cc_labels(None, None, 0, 0, None, None, None) == cc.CC_OK
    # incremental: null handle / null out
    assert lib.cc_incr_batch(None, None, 0, None, 0, None, None) == cc.CC_EINVAL
    assert lib.cc_incr_labels(None, None, None) == cc.CC_EINVAL
    assert lib.cc_incr_create(5, None, None, None) == cc.CC_EINVAL
    lib.cc_incr_destroy(None)
    assert lib.cc_incr_num_vertices(None) == 0
    assert lib.cc_workspace_bytes(1000, 5000, 2, 0) > 4000
    assert b"sm_100a" in lib.cc_version()


def test_product_has_no_cpu_fallback(monkeypatch, tmp_path):
    # a missing libcc.so must fail loudly, never fall back
    monkeypatch.setattr(cc, "_lib", None)
    monkeypatch.setattr(cc, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(cc.CCError):
        cc.load()


def test_binding_structs_mirror_header():
    """cc.py's ctypes mirrors of cc_counters / cc_opts / CC_FLAG_* follow include/cc.h."""
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "cc.h")).read(), flags=re.S)
    body = re.search(r"typedef struct\s*\{([^}]*)\}\s*cc_counters;", src).group(1)
    fields = re.findall(r"uint64_t\s+(\w+);", body)
    assert fields == list(cc.COUNTER_FIELDS)
    for name, val in re.findall(r"#define\s+CC_FLAG_(\w+)\s+\(1u\s*<<\s*(\d+)\)", src):
        assert getattr(cc, "FLAG_" + name) == 1 << int(val), name
