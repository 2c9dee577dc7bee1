"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

For every config C1..C5 the PERKS variant (bench.py's default) runs on the full domain with the same
plan bench.py uses, and its result is checked against the CPU oracle:

* C1, C2, C3, C4: the whole domain, all T steps (the oracle, multi-threaded, finishes in seconds for
  C1-C3 and in about three minutes for C4's 512^3 x 500 steps of 27 points);
* C4, C5: sampled cells, each computed by the oracle one by one on its domain of dependence: after
  T steps cell c depends only on the input within distance T of it (radius 1 stencils), so the
  oracle run on the box [c - T - 1, c + T + 1] clipped to the domain (real faces stay FRAME faces,
  the artificial box faces only corrupt cells within T of them) gives c's value exactly.  Samples
  include the frame, the faces, corners and the interior.  C4 uses T = 40 for the sampled check
  (the 27-point oracle on the full T = 500 cone would be the whole domain) plus whole-run
  properties at the full T: constant-field preservation with the dyadic preset (exact) and the
  maximum principle (values stay in [1, 2)).
Bit-exact comparison (reading R5), within the north-star tolerance as a floor.
"""
import os

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = {np.float64: 1e-12, np.float32: 1e-5}
NTHREADS = max(1, os.cpu_count() or 1)


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cfg(name):
    c = dict(si.CONFIGS[name])
    c["np_dtype"] = np.float64 if c["dtype"] == "f64" else np.float32
    return c


def _gpu_run(c, T, u0_fill=None):
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(c["stencil"])
    st = Stencil(c["shape"], offs, w, dtype=c["np_dtype"])
    if u0_fill is None:
        x = si.field_torch(c["shape"], c["np_dtype"], "cuda")
    else:
        x = torch.full(c["shape"], u0_fill, dtype=torch.float64 if c["dtype"] == "f64" else torch.float32,
                       device="cuda")
    out = torch.full_like(x, float("nan"))
    q = st.query("perks")
    st.run(x, T, "perks", out=out, workspace=st.workspace("perks"))
    torch.cuda.synchronize()
    st.close()
    return out, q


def _subbox_field(shape, lo, hi, dtype):
    """Seeded input on the box [lo, hi) of a domain of `shape` (C order), generated row by row from
    the global index (seeded_inputs is counter based), independent of the GPU path."""
    ext = [h - l for l, h in zip(lo, hi)]
    box = np.empty(ext, dtype=dtype)
    if len(shape) == 2:
        ny, nx = shape
        for j in range(ext[0]):
            box[j] = si.field((ext[1],), dtype=dtype, index_offset=(lo[0] + j) * nx + lo[1])
    else:
        nz, ny, nx = shape
        for k in range(ext[0]):
            for j in range(ext[1]):
                start = ((lo[0] + k) * ny + (lo[1] + j)) * nx + lo[2]
                box[k, j] = si.field((ext[2],), dtype=dtype, index_offset=start)
    return box


def _cone_value(c, T, cell):
    offs, w = si.preset(c["stencil"])
    shape = c["shape"]
    lo = [max(0, p - T - 1) for p in cell]
    hi = [min(n, p + T + 2) for p, n in zip(cell, shape)]
    u0 = _subbox_field(shape, lo, hi, c["np_dtype"])
    ref = oracle.run(u0, offs, w, T, nthreads=NTHREADS)
    return ref[tuple(p - l for p, l in zip(cell, lo))]


def _samples(shape, rng, n_interior=4):
    """Corners, face/frame cells, cells next to the frame and random interior cells."""
    pts = set()
    for corner in np.ndindex(*([2] * len(shape))):
        pts.add(tuple(0 if b == 0 else n - 1 for b, n in zip(corner, shape)))
    mid = tuple(n // 2 for n in shape)
    for a in range(len(shape)):
        for v in (0, 1, 2, shape[a] - 2, shape[a] - 1):
            p = list(mid)
            p[a] = v
            pts.add(tuple(p))
    for _ in range(n_interior):
        pts.add(tuple(int(rng.integers(1, n - 1)) for n in shape))
    return sorted(pts)


def _assert_close(got, ref, dtype, what):
    rel = abs(float(got) - float(ref)) / abs(float(ref))
    assert rel <= TOL[dtype], f"{what}: rel err {rel}"
    assert got == ref, f"{what}: {got!r} != {ref!r} (rel {rel})"


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_fullsize_whole_domain(name):
    _need_gpu()
    c = _cfg(name)
    T = c["steps"]
    out, q = _gpu_run(c, T)
    got = out.cpu().numpy()
    assert not np.isnan(got).any(), "unwritten (NaN) cells"
    offs, w = si.preset(c["stencil"])
    u0 = si.field(c["shape"], dtype=c["np_dtype"])
    ref = oracle.run(u0, offs, w, T, nthreads=NTHREADS)
    rel = np.max(np.abs(got.astype(np.float64) - ref) / np.abs(ref.astype(np.float64)))
    assert rel <= TOL[c["np_dtype"]], f"{name} ({q['kernel']}): max rel err {rel}"
    nbad = int(np.sum(got != ref))
    assert nbad == 0, f"{name} ({q['kernel']}): {nbad} cells differ"
    del out, got, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,T", [("C4", 40), ("C5", 100)])
def test_fullsize_sampled_cones(name, T):
    _need_gpu()
    c = _cfg(name)
    out, q = _gpu_run(c, T)
    rng = np.random.default_rng(2204)
    for cell in _samples(c["shape"], rng):
        got = out[cell].item()
        ref = _cone_value(c, T, cell)
        _assert_close(c["np_dtype"](got), ref, c["np_dtype"], f"{name} {q['kernel']} cell {cell}")
    del out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_fullsize_properties_full_T(name):
    """Whole-run properties at the full T of the bench workload: a constant field is a fixed point
    of the dyadic presets (weights sum to 1 exactly, every partial sum exact) and, for the seeded
    field, the maximum principle keeps every value in [1, 2); frame cells are bit-exact."""
    _need_gpu()
    c = _cfg(name)
    T = c["steps"]
    out, q = _gpu_run(c, T, u0_fill=1.5)
    assert bool(torch.all(out == 1.5)), f"{name} {q['kernel']}: constant field not preserved"
    del out
    out, q = _gpu_run(c, T)
    assert not bool(torch.isnan(out).any())
    assert float(out.min()) >= 1.0 and float(out.max()) < 2.0, f"{name}: maximum principle violated"
    x = si.field_torch(c["shape"], c["np_dtype"], "cuda")
    for sl in ((0,), (-1,)):
        for a in range(out.dim()):
            idx = [slice(None)] * out.dim()
            idx[a] = sl[0]
            assert bool(torch.equal(out[tuple(idx)], x[tuple(idx)])), f"{name}: frame face {a},{sl[0]} changed"
    del out, x
    torch.cuda.empty_cache()
