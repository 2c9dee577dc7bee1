"""Pins for the CG oracle (oracle/cg_oracle.c): what the paper and the mathematics fix.

SpMV (CSR): identity, hand arithmetic, exact integer/dyadic cases against a dense
numpy product (no rounding anywhere, so any correct CSR walk must agree bit for bit),
non-symmetric matrices (a transposed index fails), empty rows, and the summation error
bound against an exactly rounded row sum (math.fsum) for real-valued data.

CG (Algorithm; readings RC2-RC4): the 2x2 hand example, b = 0,
c*I in one exact step, a Poisson eigenvector in one step (closed form x = b / lambda),
n-step termination against numpy.linalg.solve, the Krylov-subspace A-norm minimisation
property computed independently by projection (a wrong sign, a swapped beta ratio or a
wrong update vector fails it), the recursive residual against b - A x_k, monotone A-norm
error, breakdown detection on indefinite matrices, and RC3 (inner products in double).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import seeded_inputs as si
import seeded_inputs.sparse as sp

DT = [np.float64, np.float32]


def _dense(row_off, col, val, n):
    a = np.zeros((n, n))
    for i in range(n):
        for k in range(row_off[i], row_off[i + 1]):
            a[i, col[k]] += val[k]
    return a


def _csr_from_dense(a):
    n = a.shape[0]
    ro, ci, va = [0], [], []
    for i in range(n):
        nz = np.nonzero(a[i])[0]
        ci.extend(nz.tolist())
        va.extend(a[i, nz].tolist())
        ro.append(len(ci))
    return np.array(ro, np.int64), np.array(ci, np.int32), np.array(va)


def _random_csr(n, m_per_row, seed, bits=None, square=True, empty_rows=()):
    """Non-symmetric random CSR (sorted columns); dyadic values if ``bits``."""
    rng = np.random.default_rng(seed)
    ro, ci, va = [0], [], []
    for i in range(n):
        k = 0 if i in empty_rows else int(rng.integers(1, m_per_row + 1))
        cols = np.sort(rng.choice(n, size=min(k, n), replace=False))
        if bits:
            vals = rng.integers(-(1 << bits), (1 << bits), size=cols.size) / float(1 << bits)
        else:
            vals = rng.standard_normal(cols.size)
        ci.extend(cols.tolist())
        va.extend(vals.tolist())
        ro.append(len(ci))
    return np.array(ro, np.int64), np.array(ci, np.int32), np.array(va)


# ------------------------------------------------------------------------------------ SpMV

@pytest.mark.parametrize("dtype", DT)
def test_spmv_identity(dtype):
    n = 37
    ro, ci, va = np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n)
    x = si.field((n,), dtype=dtype)
    assert np.array_equal(oracle.csr_spmv(ro, ci, va, x), x)


@pytest.mark.parametrize("dtype", DT)
def test_spmv_hand_2x2(dtype):
    # [[4,1],[1,3]] . [1,1] = [5,4]  (hand arithmetic)
    ro, ci, va = np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4.0, 1, 1, 3])
    y = oracle.csr_spmv(ro, ci, va, np.ones(2, dtype=dtype))
    assert y.tolist() == [5.0, 4.0]
    # and a non-symmetric one: [[0,2],[5,0]] . [3,7] = [14, 15]
    y = oracle.csr_spmv(np.array([0, 1, 2]), np.array([1, 0]), np.array([2.0, 5.0]),
                        np.array([3.0, 7.0], dtype=dtype))
    assert y.tolist() == [14.0, 15.0]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("kind", ["random", "poisson2d", "box27", "irregular"])
def test_spmv_exact_against_dense(dtype, kind):
    """Integer / dyadic matrices and 8-bit dyadic x: every product and partial sum is exact
    in the dtype, so the CSR walk must equal the dense product bit for bit."""
    if kind == "random":
        ro, ci, va = _random_csr(61, 9, seed=3, bits=6, empty_rows=(5, 17))
    elif kind == "poisson2d":
        ro, ci, va = sp.poisson2d(7, 5)
    elif kind == "box27":
        ro, ci, va = sp.box27(4)
    else:
        ro, ci, va = sp.irregular(90, mean_degree=6, heavy_rows=2, heavy_degree=40)
    n = len(ro) - 1
    x = si.field((n,), dtype=dtype, bits=8)
    y = oracle.csr_spmv(ro, ci, va, x)
    ref = _dense(ro, ci, va, n) @ x.astype(np.float64)
    assert np.array_equal(y.astype(np.float64), ref)


@pytest.mark.parametrize("dtype", DT)
def test_spmv_error_bound_real_values(dtype):
    """Real-valued data: |y_i - exact_i| <= gamma_k sum_k |a x| per row (k = row length)."""
    ro, ci, va = _random_csr(200, 30, seed=11)
    n = 200
    va = va.astype(dtype)
    x = np.random.default_rng(5).standard_normal(n).astype(dtype)
    y = oracle.csr_spmv(ro, ci, va, x)
    u = np.finfo(dtype).eps / 2
    for i in range(n):
        terms = [float(va[k]) * float(x[ci[k]]) for k in range(ro[i], ro[i + 1])]
        exact = math.fsum(terms)   # products of dtype values are exact in double for f32;
        k = len(terms)              # for f64 the product error is inside gamma_k too
        g = k * u / (1 - k * u) if k else 0.0
        assert abs(float(y[i]) - exact) <= g * math.fsum(abs(t) for t in terms) * 1.0001 + 1e-300


def test_spmv_empty_rows_and_thread_invariance():
    ro, ci, va = _random_csr(300, 12, seed=9, empty_rows=(0, 1, 150, 299))
    x = si.field((300,), dtype=np.float64)
    y1 = oracle.csr_spmv(ro, ci, va, x, nthreads=1)
    y4 = oracle.csr_spmv(ro, ci, va, x, nthreads=4)
    assert np.array_equal(y1, y4)
    assert y1[0] == 0.0 and y1[150] == 0.0 and y1[299] == 0.0


def test_spmv_rejects_bad_csr():
    with pytest.raises(oracle.OracleError):
        oracle.csr_spmv(np.array([0, 1]), np.array([3]), np.array([1.0]), np.ones(1))
    with pytest.raises(oracle.OracleError):
        oracle.csr_spmv(np.array([0, 2, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]), np.ones(3))


# -------------------------------------------------------------------------------------- CG

@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-6)])
def test_cg_hand_2x2(dtype, tol):
    # [[4,1],[1,3]] x = [1,2] -> x = [1/11, 7/11], <= 2 iterations (n-step termination)
    ro, ci, va = np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4.0, 1, 1, 3])
    x, hist, k = oracle.cg(ro, ci, va, np.array([1.0, 2.0], dtype=dtype), kmax=50,
                           tol=1e-12 if dtype == np.float64 else 1e-6)
    assert k <= 2
    assert np.allclose(x, [1 / 11, 7 / 11], rtol=0, atol=tol)
    assert hist[0] == 5.0


@pytest.mark.parametrize("dtype", DT)
def test_cg_zero_rhs_takes_no_iteration(dtype):
    ro, ci, va = sp.poisson2d(6)
    x, hist, k = oracle.cg(ro, ci, va, np.zeros(36, dtype=dtype), kmax=10, tol=0.0)
    assert k == 0 and np.all(x == 0) and hist.tolist() == [0.0]


@pytest.mark.parametrize("dtype", DT)
def test_cg_scaled_identity_one_exact_step(dtype):
    # A = 4 I: alpha = rr / (4 rr) = 1/4 exactly, x_1 = b/4, r_1 = 0 exactly, then stop (RC2)
    n = 50
    ro, ci, va = np.arange(n + 1), np.arange(n), np.full(n, 4.0)
    b = si.field((n,), dtype=dtype)
    x, hist, k = oracle.cg(ro, ci, va, b, kmax=10, tol=0.0)
    assert k == 1
    assert np.array_equal(x, (b / dtype(4)).astype(dtype))
    assert hist[1] == 0.0


@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-13), (np.float32, 1e-5)])
def test_cg_poisson_eigenvector_one_step(dtype, rtol):
    """b = sin(i pi x/(n+1)) sin(j pi y/(n+1)) is an eigenvector of the 2D Poisson matrix with
    lambda = 4 - 2cos(i pi/(n+1)) - 2cos(j pi/(n+1)) (closed form): x_1 = b / lambda and
    <r_1, r_1> ~ 0."""
    nx = 12
    ro, ci, va = sp.poisson2d(nx)
    i, j = 3, 5
    xs = np.arange(1, nx + 1)
    b = np.outer(np.sin(j * np.pi * xs / (nx + 1)), np.sin(i * np.pi * xs / (nx + 1))).ravel()
    lam = 4 - 2 * np.cos(i * np.pi / (nx + 1)) - 2 * np.cos(j * np.pi / (nx + 1))
    x, hist, k = oracle.cg(ro, ci, va, b.astype(dtype), kmax=1)
    assert k == 1
    assert np.max(np.abs(x - b / lam)) <= rtol * np.max(np.abs(b / lam)) * 10
    assert hist[1] <= (rtol * 10) ** 2 * hist[0]


def test_cg_n_step_termination_against_solve():
    rng = np.random.default_rng(4)
    n = 12
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = q @ np.diag(np.linspace(1.0, 9.0, n)) @ q.T
    a = (a + a.T) / 2
    ro, ci, va = _csr_from_dense(a)
    b = rng.standard_normal(n)
    x, hist, k = oracle.cg(ro, ci, va, b, kmax=n)
    assert k == n
    assert np.allclose(x, np.linalg.solve(a, b), rtol=0, atol=1e-10)


@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-9), (np.float32, 2e-4)])
@pytest.mark.parametrize("kind", ["poisson2d", "irregular"])
def test_cg_krylov_minimisation(dtype, rtol, kind):
    """x_k = argmin_{x in K_k(A,b)} ||x - x*||_A  (the defining property of CG): computed
    independently by projecting A onto an orthonormal basis of span{b, Ab, ..., A^{k-1} b}."""
    ro, ci, va = sp.poisson2d(8) if kind == "poisson2d" else sp.irregular(60, mean_degree=6)
    n = len(ro) - 1
    a = _dense(ro, ci, va, n)
    b = si.field((n,), dtype=dtype).astype(np.float64)
    for kk in range(1, 7):
        x, hist, k = oracle.cg(ro, ci, va, b.astype(dtype), kmax=kk)
        assert k == kk
        kry = np.empty((n, kk))
        v = b.copy()
        for m in range(kk):
            kry[:, m] = v / np.linalg.norm(v)
            v = a @ kry[:, m]
        basis, _ = np.linalg.qr(kry)
        y = np.linalg.solve(basis.T @ a @ basis, basis.T @ b)
        ref = basis @ y
        assert np.max(np.abs(x - ref)) <= rtol * np.max(np.abs(ref)), kk


@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-10), (np.float32, 1e-3)])
def test_cg_recursive_residual_and_monotone_a_norm(dtype, rtol):
    ro, ci, va = sp.poisson2d(10)
    n = len(ro) - 1
    a = _dense(ro, ci, va, n)
    b = si.field((n,), dtype=dtype)
    xstar = np.linalg.solve(a, b.astype(np.float64))
    prev = np.inf
    for kk in range(0, 25, 3):
        x, hist, k = oracle.cg(ro, ci, va, b, kmax=kk)
        res = b.astype(np.float64) - a @ x.astype(np.float64)
        assert abs(hist[-1] - res @ res) <= rtol * (b.astype(np.float64) @ b)
        e = x.astype(np.float64) - xstar
        en = e @ a @ e
        assert en <= prev * (1 + 1e-6)
        prev = en


def test_cg_inner_products_in_double():
    """RC3: <r0,r0> of an fp32 b is accumulated in double.  b_i = 1 + 2^-20 squares to a
    41-bit value; the double sum of 16 of them is exact (no float accumulation could be)."""
    n = 16
    ro, ci, va = np.arange(n + 1), np.arange(n), np.full(n, 2.0)
    b = np.full(n, 1 + 2.0 ** -20, dtype=np.float32)
    _, hist, _ = oracle.cg(ro, ci, va, b, kmax=0)
    exact = sum(Fraction(float(v)) ** 2 for v in b)
    assert Fraction(hist[0]) == exact


@pytest.mark.parametrize("dtype", DT)
def test_cg_breakdown_on_indefinite(dtype):
    # A = -I: <p, Ap> < 0 at the first step (RC4)
    n = 5
    ro, ci, va = np.arange(n + 1), np.arange(n), np.full(n, -1.0)
    with pytest.raises(oracle.OracleError) as e:
        oracle.cg(ro, ci, va, np.ones(n, dtype=dtype), kmax=3)
    assert e.value.name == "NOT_SPD"
    # diag(1,-1), b = (1,1): <p, Ap> = 0
    x, hist, k = oracle.cg(np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]),
                           np.ones(2, dtype=dtype), kmax=3, allow_not_spd=True)
    assert k == 0 and np.all(x == 0)


def test_cg_thread_count_invariance():
    ro, ci, va = sp.poisson3d(10)
    b = sp.rhs(1000)
    x1, h1, _ = oracle.cg(ro, ci, va, b, kmax=30, nthreads=1)
    x4, h4, _ = oracle.cg(ro, ci, va, b, kmax=30, nthreads=4)
    assert np.array_equal(x1, x4) and np.array_equal(h1, h4)


def test_matrices_are_symmetric_with_sorted_columns():
    for ro, ci, va in (sp.poisson2d(9, 7), sp.poisson3d(5), sp.box27(4),
                       sp.irregular(300, mean_degree=8, heavy_rows=3, heavy_degree=120)):
        n = len(ro) - 1
        a = _dense(ro, ci, va, n)
        assert np.array_equal(a, a.T)
        for i in range(n):
            c = ci[ro[i]:ro[i + 1]]
            assert np.all(np.diff(c) > 0) and i in c
        assert np.all(np.linalg.eigvalsh(a) > 0)
