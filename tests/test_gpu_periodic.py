"""GPU parity for the PERIODIC boundary (reading R1's alternative: indices wrap modulo the
extent, every cell is updated).  The general kernels (csrc/k2d_wide.cu, csrc/k3d_wide.cu) run
every point set; PERKS runs the persistent body with an empty cache split.

* small ragged domains (several tiles, partial last tile, minimum extents 2r+1): bit-exact against
  the CPU oracle's PERIODIC run (oracle.run(..., bc=BC_PERIODIC)), every preset, both dtypes,
  every variant;
* full-size domains (BASELINE.json configs C2 / C3 shapes) against the closed form of a single
  Fourier mode (PAPER.md P:204-213 written as a convolution: u0 = c0 + A cos(k.x) ->
  u_T = c0 (sum w)^T + A Re(lambda(k)^T e^{ik.x}), lambda(k) = sum_p w_p e^{i k.d_p}), within a
  rounding bound derived from the arithmetic: each step adds at most |P| u max|u| (one rounding
  per term, reading R5) and a step with positive weights summing to <= 1 does not amplify an
  earlier error, so |err_T| <= (T |P| + 1) u max|u| (+1: the rounding of u0 and of the weights).
"""
import math

import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VARIANTS = ["hostloop", "persistent", "perks", "auto"]
PRESETS_2D = ["2d5pt", "2d9pt", "2ds9pt", "2d13pt", "2d25pt", "2ds25pt"]
PRESETS_3D = ["3d7pt", "3d13pt", "3d17pt", "3d19pt", "3d27pt"]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _radius(offs):
    return max(max(abs(v) for v in o) for o in offs)


def _run_gpu(u0, offs, w, steps, variant):
    from paper_2204_02064_b200 import Stencil
    st = Stencil(u0.shape, offs, w, dtype=u0.dtype, bc="periodic")
    x = torch.from_numpy(u0).cuda()
    out = torch.full_like(x, float("nan"))
    nb = st.workspace_bytes(variant)
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device="cuda")
    ws.fill_(0xFF)
    st.run(x, steps, variant, out=out, workspace=ws)
    torch.cuda.synchronize()
    q = st.query(variant)
    st.close()
    return out.cpu().numpy(), q


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("name", PRESETS_2D + PRESETS_3D)
def test_periodic_parity_ragged(name, dtype, variant):
    _need_gpu()
    offs, w = si.preset(name)
    shape = (70, 97) if si.PRESET_NDIM[name] == 2 else (21, 37, 45)
    u0 = si.field(shape, dtype=dtype, seed=3)
    T = 7
    got, q = _run_gpu(u0, offs, w, T, variant)
    ref = oracle.run(u0, offs, w, T, bc=oracle.BC_PERIODIC)
    if q["variant"] == "perks":  # the persistent body with an empty cache split
        assert "_per" in q["kernel"] and q["cached_cells_smem"] == 0, q
    assert np.array_equal(got, ref), f"{name} {variant}: max |d| {np.nanmax(np.abs(got - ref))}"


@pytest.mark.parametrize("variant", ["hostloop", "persistent", "perks"])
@pytest.mark.parametrize("name", ["2d5pt", "2d13pt", "2ds25pt", "3d7pt", "3d13pt", "3d27pt"])
def test_periodic_minimum_extent(name, variant):
    """Extent 2r+1 on every axis: each neighbour wraps, some of them past the whole domain's
    width minus one (the single-wrap case the kernels rely on)."""
    _need_gpu()
    offs, w = si.preset(name)
    r = _radius(offs)
    nd = si.PRESET_NDIM[name]
    shape = (2 * r + 1,) * nd
    u0 = si.field(shape, dtype=np.float64, seed=9)
    got, _ = _run_gpu(u0, offs, w, 5, variant)
    assert np.array_equal(got, oracle.run(u0, offs, w, 5, bc=oracle.BC_PERIODIC))


@pytest.mark.parametrize("variant", ["hostloop", "persistent", "perks"])
@pytest.mark.parametrize("ndim", [2, 3])
def test_periodic_random_nonsymmetric_weights(ndim, variant):
    """Non-symmetric weights: a mirrored offset or a wrap in the wrong direction changes the
    result (the Fourier symbol becomes complex)."""
    _need_gpu()
    offs, _ = si.preset("2d9pt" if ndim == 2 else "3d27pt")
    w = si.random_convex_weights(len(offs), np.float32, seed=21)
    shape = (53, 140) if ndim == 2 else (19, 23, 66)
    u0 = si.field(shape, dtype=np.float32, seed=4)
    got, _ = _run_gpu(u0, offs, w, 9, variant)
    assert np.array_equal(got, oracle.run(u0, offs, w, 9, bc=oracle.BC_PERIODIC))


def _fourier_case(shape, offs, w, m, dtype, T, c0=1.25, A=0.5):
    nd = len(shape)
    ext = tuple(reversed(shape))  # (nx, ny[, nz])
    k = tuple(2 * math.pi * m[a] / ext[a] for a in range(nd))
    grids = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")  # (z,) y, x
    coords = list(reversed(grids))  # x, y[, z]
    phase = sum(k[a] * coords[a] for a in range(nd))
    u0 = (c0 + A * np.cos(phase)).astype(dtype)
    wq = [float(np.asarray(v, dtype=dtype)) for v in w]  # reading R6: weights rounded once
    lam = sum(wp * np.exp(1j * sum(k[a] * o[a] for a in range(nd))) for wp, o in zip(wq, offs))
    exact = c0 * sum(wq) ** T + A * np.real(lam ** T * np.exp(1j * phase))
    u = np.finfo(dtype).eps / 2
    bound = (T * len(offs) + 1) * u * (c0 + A) * 2  # x2: the u0 rounding and cos() itself
    return u0, exact, bound


@pytest.mark.parametrize("variant", ["hostloop", "persistent", "perks"])
@pytest.mark.parametrize("case", ["C2_2d9pt_f32", "C3_3d7pt_f64"])
def test_periodic_fourier_full_size(case, variant):
    _need_gpu()
    if case.startswith("C2"):
        name, shape, dtype, T, m = "2d9pt", (3072, 3072), np.float32, 1000, (3, 2)
    else:
        name, shape, dtype, T, m = "3d7pt", (256, 256, 256), np.float64, 1000, (2, 1, 3)
    offs, w = si.preset(name)
    u0, exact, bound = _fourier_case(shape, offs, w, m, dtype, T)
    got, _ = _run_gpu(u0, offs, w, T, variant)
    err = np.max(np.abs(got.astype(np.float64) - exact))
    # the decayed mode is still far above the bound: a wrong wrap would show
    amp = np.max(np.abs(exact - np.mean(exact)))
    assert amp > 100 * bound
    assert err <= bound, f"max |err| {err:.3e} > bound {bound:.3e}"
