"""GPU parity of the two-steps-per-pass PERKS-3D kernel (k3d_tb.cu, reading R13): level
t+1 of the planes in flight is kept in shared memory and level t+2 stored, with a redundant ring of
level t+1 around each tile computed by the halo warps.  Bit-exact against the oracle (reading R5)
for every r = 1 3D shape and dtype, odd and even T (odd T: one single-step pass first), ragged
tiles and z chunks, several units per CTA (few SMs), both traversal orders, back-to-back runs.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

from test_gpu_parity import _check, _need_gpu, _run_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SHAPES = [(3, 9, 8), (3, 20, 64), (5, 7, 16), (9, 17, 36), (34, 40, 132), (37, 24, 128), (64, 48, 100)]


def _kernel(name, shape, dtype):
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=dtype)
    q = st.query("perks")
    st.close()
    return q


@pytest.mark.parametrize("name", ["3d7pt", "3d27pt", "3d19pt"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", SHAPES)
def test_tb3d_parity(monkeypatch, name, dtype, shape):
    _need_gpu()
    monkeypatch.setenv("PERKS_P3D_TB", "1")
    q = _kernel(name, shape, dtype)
    assert q["kernel"].startswith("perks3d_tb2"), q
    u0 = si.field(shape, dtype=dtype, seed=808)
    offs, w = si.preset(name)
    for T in (1, 2, 3, 8):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


@pytest.mark.parametrize("nsm,nzc,zigzag,rng", [("3", "0", "1", "0"), ("5", "7", "0", "0"), ("2", "3", "1", "0"),
                                              ("0", "11", "1", "0"), ("3", "0", "1", "1"), ("7", "0", "0", "1"),
                                              ("0", "0", "1", "1"), ("13", "0", "1", "1")])
@pytest.mark.parametrize("name,dtype", [("3d7pt", np.float64), ("3d27pt", np.float32), ("3d19pt", np.float64)])
def test_tb3d_units_and_chunks(monkeypatch, nsm, nzc, zigzag, rng, name, dtype):
    """Several units per CTA (PERKS_NUM_SMS), forced z chunking, zig-zag on/off; balanced contiguous
    runs of (tile, plane) split at tile boundaries (PERKS_TB_RANGE=1), also over several tiles."""
    _need_gpu()
    monkeypatch.setenv("PERKS_P3D_TB", "1")
    if nsm != "0":
        monkeypatch.setenv("PERKS_NUM_SMS", nsm)
    monkeypatch.setenv("PERKS_TB_NZC", nzc)
    monkeypatch.setenv("PERKS_ZIGZAG", zigzag)
    monkeypatch.setenv("PERKS_TB_RANGE", rng)
    shape = (45, 50, 136)
    assert _kernel(name, shape, dtype)["kernel"].startswith("perks3d_tb2")
    u0 = si.field(shape, dtype=dtype, seed=909)
    offs, w = si.preset(name)
    for T in (4, 7):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_tb3d_random_weights_and_default(dtype):
    """Random (non-symmetric) convex weights; the 7-point star takes this kernel by default (AUTO and PERKS)."""
    _need_gpu()
    shape = (30, 33, 72)
    q = _kernel("3d7pt", shape, dtype)
    assert q["kernel"].startswith("perks3d_tb2"), q
    offs, _ = si.preset("3d7pt")
    w = si.random_convex_weights(len(offs), dtype, seed=17)
    u0 = si.field(shape, dtype=dtype, seed=1001)
    for T in (5, 6):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        _check(_run_gpu(u0, "3d7pt", w, T, "perks"), ref, u0, dtype)
        _check(_run_gpu(u0, "3d7pt", w, T, "auto"), ref, u0, dtype)


def test_tb3d_grid_barrier_counter_wrap(monkeypatch):
    """The pass barrier's 32-bit counter wraps mid-run (started 700 below 2^32; 96 CTAs x 11 pass
    barriers) and the two-steps-per-pass run stays bit-exact."""
    _need_gpu()
    monkeypatch.setenv("PERKS_TEST_BAR_BASE", str(2**32 - 700))
    shape = (64, 96, 128)
    q = _kernel("3d7pt", shape, np.float64)
    assert q["kernel"].startswith("perks3d_tb2") and q["grid"] * 11 > 700, q
    u0 = si.field(shape, dtype=np.float64, seed=1111)
    offs, w = si.preset("3d7pt")
    ref = oracle.run(u0, offs, w, 24, nthreads=8)
    _check(_run_gpu(u0, "3d7pt", w, 24, "perks"), ref, u0, np.float64)
