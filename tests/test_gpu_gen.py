"""The CUDA input generator (inputs/libccgen.so) reproduces inputs/gen.py byte for byte."""
import numpy as np
import pytest

from inputs import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from inputs import gpu as ggen  # noqa: E402


def same(d, h):
    d_off, d_adj = d
    off, adj = h
    assert np.array_equal(d_off.cpu().numpy(), off)
    assert np.array_equal(d_adj.cpu().numpy().view(np.uint32), adj)


def test_er_c1_bytes():
    same(ggen.er(1), gen.er(1))
    same(ggen.er(9, n0=777, pairs=1500, isolated=3), gen.er(9, n0=777, pairs=1500, isolated=3))


def test_grid_bytes():
    same(ggen.grid(2, 256, 300), gen.grid(2, 256, 300))
    same(ggen.grid(3, 17, 5, p32=1 << 32), gen.grid(3, 17, 5, p32=1 << 32))


@pytest.mark.parametrize("scale", [6, 12, 16])
def test_rmat_bytes(scale):
    same(ggen.rmat(3, scale), gen.rmat(3, scale))
    same(ggen.rmat(4, scale, permuted=False), gen.rmat(4, scale, permuted=False))


def test_incr_batches_bytes():
    for b in (0, 1, 37):
        ins, qs = ggen.incr_batch(5, 14, b, 1000, 111)
        hi, hq = gen.incr_batch(5, 14, b, 1000, 111)
        assert np.array_equal(ins.cpu().numpy().view(np.uint32), hi)
        assert np.array_equal(qs.cpu().numpy().view(np.uint32), hq)


@pytest.mark.parametrize("scale", [10, 16])
def test_exp_weights_bytes(scale):
    off, adj = gen.rmat(3, scale)
    d_off, d_adj = ggen.rmat(3, scale)
    w = ggen.exp_weights(d_off, d_adj, 3)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), gen.exp_weights(off, adj, 3).view(np.uint32))
    go, ga = ggen.grid(2, 64, 70)
    ho, ha = gen.grid(2, 64, 70)
    assert np.array_equal(ggen.exp_weights(go, ga, 11).cpu().numpy().view(np.uint32),
                          gen.exp_weights(ho, ha, 11).view(np.uint32))


def test_rm_stream_bytes():
    """The Table 4 RM stream (a,b,c = .5,.1,.1, unpermuted) equals gen.rmat_pairs."""
    for s, first, count, perm in ((10, 0, 5000, False), (30, 123456, 4096, False), (20, 7, 3000, True)):
        d = ggen.rmat_stream(3, s, first, count, permuted=perm).cpu().numpy().view(np.uint32)
        u, v = gen.rmat_pairs(3, s, first, count, permuted=perm, t=gen.RM_T)
        assert np.array_equal(d[:, 0], u.astype(np.uint32)) and np.array_equal(d[:, 1], v.astype(np.uint32))
