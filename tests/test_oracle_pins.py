"""Pins for the CPU oracle (oracle/): things the paper and the mathematics fix.

Each test checks the oracle against something other than itself:
closed forms (identity, shift, constant, single Fourier mode), an independent
exact-rational evaluator (tests/exact_rational.py), and invariants (linearity,
composability, maximum principle, mass conservation).  A plausible mistake in
the oracle (dropped term, wrong sign/axis, frame off-by-one, wrong weight to a
neighbour, wrong step count/parity) fails at least one of them.

Citations: Eq. iterativeStencil P:204-213 (operator and orientation),
P:182-193 (out-of-place iteration), SPEC S:387-404 / S:426 (test ideas).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import seeded_inputs as si
from exact_rational import run_exact

DT = [np.float64, np.float32]


def _rand_field(shape, dtype, seed=1):
    return si.field(shape, dtype=dtype, seed=seed)


# ------------------------------------------------------------ identity / T=0

@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("bc", [oracle.BC_FRAME, oracle.BC_PERIODIC])
@pytest.mark.parametrize("shape", [(7, 9), (5, 6, 7)])
def test_identity_and_T0(dtype, bc, shape):
    u = _rand_field(shape, dtype)
    # single point (0,0,0), w=1: out == in exactly, any T
    for T in (0, 1, 4):
        out = oracle.run(u, [(0, 0, 0)], [1.0], T, bc=bc)
        assert np.array_equal(out, u)
    # T=0 returns the input for any stencil
    offs, w = si.preset("2d9pt" if len(shape) == 2 else "3d27pt")
    assert np.array_equal(oracle.run(u, offs, w, 0, bc=bc), u)


# ------------------------------------------------------------ shift closed form

@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("axis,sign", [(0, 1), (0, -1), (1, 1), (1, -1), (2, 1), (2, -1)])
def test_shift_closed_form(dtype, axis, sign):
    """Single point d = sign*e_axis, w=1 (orientation P:207-208: E = i+1 = x+1).

    PERIODIC: out[c] = in[c + T*d mod n].
    FRAME (r=1): interior out[c] = in[clamp(c_axis + T*sign, 0, n-1)], frame unchanged.
    """
    shape = (6, 7, 9)  # (nz, ny, nx)
    u = _rand_field(shape, dtype, seed=3)
    d = [0, 0, 0]
    d[axis] = sign
    np_axis = 2 - axis  # x is the last numpy axis
    for T in (1, 2, 5):
        per = oracle.run(u, [tuple(d)], [1.0], T, bc=oracle.BC_PERIODIC)
        assert np.array_equal(per, np.roll(u, -sign * T, axis=np_axis))
        fr = oracle.run(u, [tuple(d)], [1.0], T, bc=oracle.BC_FRAME)
        exp = u.copy()
        n = shape[np_axis]
        interior = (slice(1, -1),) * 3
        idx = np.arange(n)
        src = np.clip(idx + sign * T, 0, n - 1)
        shifted = np.take(u, src, axis=np_axis)
        exp[interior] = shifted[interior]
        assert np.array_equal(fr, exp)


# ------------------------------------------------------------ constant fixed point

@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("name", ["2d5pt", "2d9pt", "3d7pt", "3d27pt", "3d19pt", "2ds9pt", "2d13pt",
                                  "2d17pt", "2d21pt", "2ds25pt", "2d25pt", "3d13pt", "3d17pt"])
@pytest.mark.parametrize("bc", [oracle.BC_FRAME, oracle.BC_PERIODIC])
def test_constant_preserved(dtype, name, bc):
    """Dyadic presets sum to exactly 1 -> a constant field is a fixed point."""
    offs, w = si.preset(name)
    assert sum(Fraction(x) for x in w) == 1
    shape = (15, 17) if si.PRESET_NDIM[name] == 2 else (5, 6, 7)  # >= 2r+1 (r <= 6 in 2D, 2 in 3D)
    u = np.full(shape, 1.5, dtype=dtype)
    out = oracle.run(u, offs, w, 13, bc=bc)
    assert np.all(out == dtype(1.5))


# ------------------------------------------------------------ Fourier mode

def _lambda_hat(offs, w, k):
    return sum(wp * np.exp(1j * (k[0] * d[0] + k[1] * d[1] + k[2] * d[2]))
               for d, wp in zip(offs, w))


@pytest.mark.parametrize("name", ["2d5pt", "2d9pt", "3d7pt", "3d27pt", "3d19pt", "2ds9pt", "2d13pt",
                                  "2ds25pt", "2d25pt", "3d13pt", "3d17pt", "rand2d", "rand3d"])
def test_fourier_mode_decay(name):
    """PERIODIC: u0 = c0 + A·cos(k·x) -> u_T = c0·(Σw)^T + A·Re(λ̂(k)^T e^{ik·x}),
    λ̂(k) = Σ_p w_p e^{i k·d_p}.  Non-symmetric random weights make λ̂ complex, which
    pins the sign/orientation of every offset (a mirrored offset conjugates λ̂)."""
    if name.startswith("rand"):
        base = "2d9pt" if name == "rand2d" else "3d27pt"
        offs, _ = si.preset(base)
        w = si.random_convex_weights(len(offs), np.float64, seed=11)
    else:
        offs, w = si.preset(name)
    ndim = 2 if ("2d" in name) else 3
    if ndim == 2:
        nx, ny, nz = 24, 20, 1
        m = (3, 2, 0)
    else:
        nx, ny, nz = 12, 10, 8
        m = (2, 1, 3)
    k = (2 * math.pi * m[0] / nx, 2 * math.pi * m[1] / ny, 2 * math.pi * m[2] / nz)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    phase = k[0] * x + k[1] * y + k[2] * z
    c0, A = 1.25, 0.5
    u0 = c0 + A * np.cos(phase)
    if ndim == 2:
        u0 = u0[0]
        phase = phase[0]
    T = 40
    out = oracle.run(np.ascontiguousarray(u0), offs, w, T, bc=oracle.BC_PERIODIC)
    lam = _lambda_hat(offs, w, k)
    s = sum(w)
    exact = c0 * s ** T + A * np.real(lam ** T * np.exp(1j * phase))
    tol = 8 * T * len(offs) * np.finfo(np.float64).eps * 2.0
    assert np.max(np.abs(out - exact)) < tol


# ------------------------------------------------------------ exact rational

def _dyadic_field(shape, dtype):
    return si.field(shape, dtype=dtype, bits=10, seed=5)


# (name, fp64 window, fp32 window) — the last T at which a plain run is still
# exact (SURVEY Appendix C for the r = 1 presets; the rest measured with
# tests/exact_rational.py on the grids of _exact_shape, re-checked below).
WINDOWS = {"2d5pt": (14, 4), "2d9pt": (10, 3), "3d7pt": (14, 4), "3d27pt": (7, 2),
           "3d19pt": (8, 2), "2ds9pt": (10, 3), "2d13pt": (8, 2), "2d17pt": (7, 2),
           "2d21pt": (6, 1), "2ds25pt": (5, 1), "2d25pt": (5, 1), "3d13pt": (8, 2), "3d17pt": (7, 2)}


def _exact_shape(name):
    """Tiny grids whose FRAME interior (width r = the preset's radius, reading R1) is at least
    2r cells wide, so a wrong frame width or a wrong offset reach changes interior cells."""
    offs, _ = si.preset(name)
    r = max(max(abs(d) for d in o) for o in offs)
    if si.PRESET_NDIM[name] == 2:
        return (8, 8) if r == 1 else (4 * r + 4, 4 * r + 4)
    return (6, 6, 6) if r == 1 else (2 * r + 4,) * 3


def _representable(v: Fraction, dtype) -> bool:
    f = dtype(float(v))
    return Fraction(float(f)) == v


@pytest.mark.parametrize("name", sorted(WINDOWS))
@pytest.mark.parametrize("bc", [oracle.BC_FRAME, oracle.BC_PERIODIC])
@pytest.mark.parametrize("dtype", DT)
def test_exact_rational_window(name, bc, dtype):
    """Inside the exactness window the oracle equals exact rational arithmetic bit for bit
    (every Table II preset, radius 1-6: pins the FRAME width r and the offset reach)."""
    offs, w = si.preset(name)
    shape = _exact_shape(name)
    dims = (shape[-1], shape[-2], shape[0] if len(shape) == 3 else 1)
    u = _dyadic_field(shape, dtype)
    exact = [Fraction(float(v)) for v in u.ravel()]
    win = WINDOWS[name][0 if dtype == np.float64 else 1]
    cur = exact
    last_exact = 0
    for T in range(1, win + 1):
        cur = run_exact(cur, dims, offs, w, 1, periodic=(bc == oracle.BC_PERIODIC))
        if not all(_representable(v, dtype) for v in cur):
            break
        last_exact = T
        out = oracle.run(u, offs, w, T, bc=bc)
        assert [Fraction(float(v)) for v in out.ravel()] == cur, f"T={T}"
    assert last_exact >= win


@pytest.mark.parametrize("name", ["2d5pt", "3d7pt", "2d9pt"])
@pytest.mark.parametrize("dtype", DT)
def test_exact_rational_random_weights(name, dtype):
    """Non-symmetric random weights: |oracle - exact| within the fma error bound.

    The exact evaluator uses the dtype-rounded weights (reading R6), so any
    misplaced weight/neighbour shows as an O(1e-2) error, far above the bound.
    """
    offs, _ = si.preset(name)
    w = si.random_convex_weights(len(offs), dtype, seed=17)
    shape = (8, 9) if si.PRESET_NDIM[name] == 2 else (5, 6, 7)
    dims = (shape[-1], shape[-2], shape[0] if len(shape) == 3 else 1)
    u = _rand_field(shape, dtype, seed=9)
    T = 6
    exact = run_exact([Fraction(float(v)) for v in u.ravel()], dims, offs,
                      [float(x) for x in w], T)
    out = oracle.run(u, offs, w, T)
    err = max(abs(float(Fraction(float(a)) - b)) for a, b in zip(out.ravel(), exact))
    u_eps = np.finfo(dtype).eps
    assert err <= 2 * T * len(offs) * u_eps * 2.0
    assert err < 1e-3


# ------------------------------------------------------------ invariants

@pytest.mark.parametrize("dtype", DT)
def test_linearity(dtype):
    offs, _ = si.preset("3d7pt")
    w = si.random_convex_weights(len(offs), dtype, seed=2)
    u = _rand_field((6, 7, 8), np.float64, seed=21).astype(dtype)
    v = _rand_field((6, 7, 8), np.float64, seed=22).astype(dtype)
    a, b = dtype(0.75), dtype(-0.5)
    T = 10
    lhs = oracle.run((a * u + b * v).astype(dtype), offs, w, T, bc=oracle.BC_PERIODIC)
    rhs = a * oracle.run(u, offs, w, T, bc=oracle.BC_PERIODIC) + b * oracle.run(
        v, offs, w, T, bc=oracle.BC_PERIODIC)
    tol = 4 * T * len(offs) * np.finfo(dtype).eps * 2
    assert np.max(np.abs(lhs.astype(np.float64) - rhs.astype(np.float64))) < tol


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("name", ["2d5pt", "2d9pt", "3d7pt", "3d27pt", "3d19pt"])
def test_composability(dtype, name):
    """run(T1) then run(T2) == run(T1+T2) bit-exact (the iteration is Markov)."""
    offs, w = si.preset(name)
    shape = (13, 17) if si.PRESET_NDIM[name] == 2 else (7, 8, 9)
    u = _rand_field(shape, dtype, seed=4)
    a = oracle.run(oracle.run(u, offs, w, 3), offs, w, 4)
    b = oracle.run(u, offs, w, 7)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", DT)
def test_maximum_principle_and_frame(dtype):
    offs, _ = si.preset("2d9pt")
    w = si.random_convex_weights(len(offs), dtype, seed=5)
    u = _rand_field((31, 29), dtype, seed=6)
    out = oracle.run(u, offs, w, 25)
    slack = 50 * np.finfo(dtype).eps * 2
    assert out.min() >= u.min() - slack and out.max() <= u.max() + slack
    # frame cells are bit-exact copies of the input
    assert np.array_equal(out[0, :], u[0, :]) and np.array_equal(out[-1, :], u[-1, :])
    assert np.array_equal(out[:, 0], u[:, 0]) and np.array_equal(out[:, -1], u[:, -1])
    # and interior cells did change
    assert not np.array_equal(out[1:-1, 1:-1], u[1:-1, 1:-1])


def test_mass_conservation_periodic():
    offs, w = si.preset("3d27pt")
    u = _rand_field((6, 8, 10), np.float64, seed=8)
    out = oracle.run(u, offs, w, 30, bc=oracle.BC_PERIODIC)
    assert abs(out.sum() - u.sum()) < 1e-10 * u.size


def test_threads_bit_identical():
    offs, w = si.preset("3d27pt")
    u = _rand_field((10, 12, 14), np.float32, seed=12)
    a = oracle.run(u, offs, w, 9, nthreads=1)
    b = oracle.run(u, offs, w, 9, nthreads=4)
    assert np.array_equal(a, b)


# ------------------------------------------------------------ errors

def test_invalid_domain():
    offs, w = si.preset("2d5pt")
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(np.ones((2, 5)), offs, w, 1)
    assert e.value.name == "INVALID_DOMAIN"
    # the minimum legal extent is 2r+1 = 3
    oracle.run(np.ones((3, 3)), offs, w, 1)


def test_generator_torch_matches_numpy():
    torch = pytest.importorskip("torch")
    for dt in (np.float32, np.float64):
        a = si.field((3, 5, 7), dtype=dt, index_offset=1000)
        b = si.field_torch((3, 5, 7), dt, "cpu", index_offset=1000).numpy()
        assert np.array_equal(a, b)
    # slab generation equals the global field
    g = si.field((8, 4, 4), np.float64)
    s = si.field((4, 4, 4), np.float64, index_offset=4 * 16)
    assert np.array_equal(g[4:], s)


# ------------------------------------------------------------ rounding order

def _round_frac(v: Fraction, mant_bits: int) -> Fraction:
    """Correctly round a rational to the nearest binary float with mant_bits
    significand bits (round half to even); normal range only."""
    if v == 0:
        return Fraction(0)
    sign = -1 if v < 0 else 1
    a = abs(v)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    scale = Fraction(2) ** (mant_bits - 1 - e)
    q = a * scale
    n, r = divmod(q.numerator, q.denominator)
    rem = Fraction(r, q.denominator)
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * Fraction(n) / scale


@pytest.mark.parametrize("dtype,mbits", [(np.float64, 53), (np.float32, 24)])
def test_fma_chain_rounding(dtype, mbits):
    """Reading R5: acc = RN(w0·v0); acc = RN(w_p·v_p + acc) for p = 1.. in list order
    (a single rounding per fused multiply-add).  Pinned against exact rationals with
    explicit correct rounding, so a non-fused chain or a reordered sum fails."""
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0)]
    w = [float(x) for x in np.array([0.3, 0.7 / 3, 0.1, 0.2], dtype=dtype)]
    u = _rand_field((5, 9), dtype, seed=31)
    out = oracle.run(u, offs, w, 1, bc=oracle.BC_PERIODIC)
    ny, nx = u.shape
    bad = 0
    for y in range(ny):
        for x in range(nx):
            acc = None
            for (dx, dy, _), wp in zip(offs, w):
                v = Fraction(float(u[(y + dy) % ny, (x + dx) % nx]))
                term = Fraction(wp) * v
                acc = _round_frac(term if acc is None else term + acc, mbits)
            bad += Fraction(float(out[y, x])) != acc
    assert bad == 0
