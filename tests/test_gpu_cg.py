"""GPU parity for the PERKS CG solver (NEXT-3) through the C ABI (include/perks/perks_cg.h).

What must match (readings RC1-RC5):
* SpMV: on integer / dyadic data every product and partial sum is exact in any order, so the
  merge-based SpMV must equal the oracle's row-order sum bit for bit (incl. empty rows, rows
  split across threads, tiles and a row longer than a whole tile).  On real-valued data both
  sides are within gamma_k * sum |a x| of the exact row sum, so they differ by at most twice
  that (RC1).
* CG: the iterates differ from the oracle only by the summation order of the SpMV rows and the
  inner products; the tolerance is RC5's (measured reorder sensitivity x 100).
* Variants (host loop / persistent / PERKS) and cache policies (IMP / VEC / MAT / MIX) share
  the partition and the reduction order: bit-identical x, history and iteration count.
Outputs are NaN-poisoned before every run so an unwritten entry cannot pass.
"""
import math

import numpy as np
import pytest

import oracle
import seeded_inputs as si
import seeded_inputs.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DT = [np.float64, np.float32]
# RC5: the GPU may differ from the oracle by at most SPREAD_FACTOR x the oracle's own spread
# under reorderings of the same problem (symmetric permutations P A P^T, P b: identical
# mathematics, different summation orders; the largest deviation over N_PERM of them), plus a
# floor of a few ulps of the result.
SPREAD_FACTOR = 30.0
N_PERM = 4
# fixed-size parity (full workloads) where the permuted oracle would take too long:
XTOL = {np.float64: 1e-9, np.float32: 2e-3}
RTOL_HIST = {np.float64: 1e-6, np.float32: 5e-2}
POLICIES = [("hostloop", "imp"), ("persistent", "imp"), ("perks", "vec"), ("perks", "mat"), ("perks", "mix")]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cg(ro, ci, va, dtype):
    from paper_2204_02064_b200 import CG
    return CG(ro, ci, va, dtype="f64" if dtype == np.float64 else "f32")


def _gpu_spmv(h, x):
    xt = torch.from_numpy(x).cuda()
    y = torch.full_like(xt, float("nan"))
    h.spmv(xt, out=y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _gpu_solve(h, b, kmax, tol=0.0, variant="perks", policy="auto"):
    bt = torch.from_numpy(b).cuda()
    x = torch.full_like(bt, float("nan"))
    ws = h.workspace()
    ws.fill_(0xFF)
    x, hist, info = h.solve(bt, kmax, tol, variant, policy, out=x)
    torch.cuda.synchronize()
    return x.cpu().numpy(), hist.cpu().numpy(), info.cpu().numpy()


def _long_row_matrix(n=3000, long_len=9000):
    """Diagonal + one row/column pair far longer than a tile (NT*IPT path items): the row is
    split across many threads AND several tiles of its CTA."""
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.full(n, float(n))]
    j = np.unique(np.linspace(0, n - 1, num=min(long_len, n)).astype(np.int64))
    j = j[j != 7]
    rows += [np.full(j.size, 7), j]
    cols += [j, np.full(j.size, 7)]
    vals += [np.full(j.size, -0.5), np.full(j.size, -0.5)]
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    o = np.lexsort((c, r))
    r, c, v = r[o], c[o], v[o]
    ro = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=ro[1:])
    return ro, c.astype(np.int32), v


def _dense_long_rows(n=400):
    """Every row dense (n nonzeros): rows longer than a thread's slice everywhere."""
    rng = np.random.default_rng(2)
    a = rng.integers(-8, 8, size=(n, n)).astype(np.float64)
    ro = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    return ro, ci, a.ravel()


def _random_csr(n, m, seed, empty_rows=()):
    rng = np.random.default_rng(seed)
    ro, ci, va = [0], [], []
    for i in range(n):
        k = 0 if i in empty_rows else int(rng.integers(1, m + 1))
        c = np.sort(rng.choice(n, size=min(k, n), replace=False))
        ci.extend(c.tolist())
        va.extend((rng.integers(-64, 64, size=c.size) / 64.0).tolist())
        ro.append(len(ci))
    return np.array(ro, np.int64), np.array(ci, np.int32), np.array(va)


SPMV_MATS = {
    "poisson2d_37x23": lambda: sp.poisson2d(37, 23),
    "poisson3d_20": lambda: sp.poisson3d(20),
    "box27_14": lambda: sp.box27(14),
    "irregular_5000": lambda: sp.irregular(5000, mean_degree=10, heavy_rows=4, heavy_degree=600),
    "random_empty_rows": lambda: _random_csr(4000, 12, 3, empty_rows=(0, 1, 2, 1999, 3999)),
    "long_row": _long_row_matrix,
    "dense_rows": _dense_long_rows,
    "tiny_1x1": lambda: (np.array([0, 1]), np.array([0], np.int32), np.array([3.0])),
    "tiny_2x2": lambda: (np.array([0, 2, 4]), np.array([0, 1, 0, 1], np.int32), np.array([4.0, 1, 1, 3])),
}


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("name", list(SPMV_MATS))
def test_spmv_bit_exact_on_exact_data(name, dtype):
    _need_gpu()
    ro, ci, va = SPMV_MATS[name]()
    n = len(ro) - 1
    x = si.field((n,), dtype=dtype, bits=8)
    h = _cg(ro, ci, va, dtype)
    y = _gpu_spmv(h, x)
    ref = oracle.csr_spmv(ro, ci, va, x)
    assert np.array_equal(y, ref), f"{int(np.sum(y != ref))} rows differ"
    h.close()


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("name", ["irregular_5000", "long_row", "box27_14", "dense_rows"])
def test_spmv_real_values_within_reorder_bound(name, dtype):
    _need_gpu()
    ro, ci, va = SPMV_MATS[name]()
    rng = np.random.default_rng(8)
    va = (va * rng.uniform(0.5, 1.5, size=va.shape)).astype(dtype).astype(np.float64)
    n = len(ro) - 1
    x = rng.standard_normal(n).astype(dtype)
    h = _cg(ro, ci, va, dtype)
    y = _gpu_spmv(h, x).astype(np.float64)
    ref = oracle.csr_spmv(ro, ci, va, x).astype(np.float64)
    u = np.finfo(dtype).eps / 2
    k = np.diff(ro).astype(np.float64) + 1
    absprod = np.abs(va.astype(dtype).astype(np.float64)) * np.abs(x.astype(np.float64)[ci])
    s = np.add.reduceat(np.concatenate([absprod, [0.0]]), np.minimum(ro[:-1], len(absprod)))
    s[np.diff(ro) == 0] = 0.0
    bound = 2 * (k * u / (1 - k * u)) * s
    assert np.all(np.abs(y - ref) <= bound * 1.0001 + 1e-300)
    h.close()


def test_partition_is_row_aligned_and_balanced():
    _need_gpu()
    ro, ci, va = sp.irregular(200000)
    from paper_2204_02064_b200 import CG
    h = CG(ro, ci, va)
    rows = h.partition()
    n, nnz = len(ro) - 1, len(ci)
    assert rows[0] == 0 and rows[-1] == n and np.all(np.diff(rows) >= 0)
    g = len(rows) - 1
    path = np.diff(rows + ro[rows])
    assert path.max() <= (n + nnz) / g + np.diff(ro).max() + 1
    h.close()


def _permuted(ro, ci, va, b, seed):
    n = len(ro) - 1
    perm = np.random.default_rng(seed).permutation(n)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rows, cols, vals = [], [], []
    for i2, i in enumerate(perm):
        c = inv[ci[ro[i]:ro[i + 1]]]
        o = np.argsort(c)
        rows.append(np.full(c.size, i2))
        cols.append(c[o])
        vals.append(va[ro[i]:ro[i + 1]][o])
    ro2 = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=ro2[1:])
    return perm, ro2, np.concatenate(cols).astype(np.int32), np.concatenate(vals), b[perm]


def _oracle_spread(ro, ci, va, b, K):
    """(x_ref, hist_ref, x_spread, res_spread): the oracle's own deviation under two symmetric
    permutations (RC5), as max|dx| / max|x| and max_k |sqrt(h_k) - sqrt(h'_k)| / sqrt(h_0)."""
    xo, ho, ko = oracle.cg(ro, ci, va, b, kmax=K)
    xs = rs = 0.0
    for seed in range(1, N_PERM + 1):
        perm, ro2, ci2, va2, b2 = _permuted(ro, ci, va, b, seed)
        x2, h2, k2 = oracle.cg(ro2, ci2, va2, b2, kmax=K)
        assert k2 == ko
        xu = np.empty_like(x2)
        xu[perm] = x2
        xs = max(xs, np.max(np.abs(xu.astype(np.float64) - xo)) / np.max(np.abs(xo)))
        rs = max(rs, np.max(np.abs(np.sqrt(h2) - np.sqrt(ho))) / np.sqrt(ho[0]))
    return xo, ho, ko, xs, rs


def _k_before_floor(ro, ci, va, b, K, dtype):
    """Largest K' <= K whose <r,r> stays above the rounding floor (so the iteration count is
    deterministic: no run stops early on an exact zero)."""
    _, ho, ko = oracle.cg(ro, ci, va, b, kmax=K)
    floor = 1e-24 if dtype == np.float64 else 1e-10
    ok = np.nonzero(ho / ho[0] < floor)[0]
    return int(min(ko, ok[0] - 1 if ok.size else K))


CG_MATS = {
    "poisson2d_40": lambda: sp.poisson2d(40),
    "poisson3d_14": lambda: sp.poisson3d(14),
    "box27_12": lambda: sp.box27(12),
    "irregular_3000": lambda: sp.irregular(3000, mean_degree=8, heavy_rows=3, heavy_degree=300),
    "long_row": _long_row_matrix,
}


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("name", list(CG_MATS))
def test_cg_matches_oracle_and_all_variants_identical(name, dtype):
    _need_gpu()
    ro, ci, va = CG_MATS[name]()
    n = len(ro) - 1
    b = sp.rhs(n, dtype=dtype)
    K = _k_before_floor(ro, ci, va, b, 40, dtype)
    assert K >= 2
    xo, ho, ko, xs, rs = _oracle_spread(ro, ci, va, b, K)
    eps = np.finfo(dtype).eps
    h = _cg(ro, ci, va, dtype)
    ref = None
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, b, K, 0.0, variant, policy)
        assert not np.isnan(x).any()
        assert info.tolist() == [ko, 0]
        if ref is None:
            ref = (x, hist)
            err = np.max(np.abs(x.astype(np.float64) - xo)) / np.max(np.abs(xo))
            assert err <= SPREAD_FACTOR * xs + 8 * eps, f"x rel err {err:.3g} vs oracle spread {xs:.3g}"
            rerr = np.max(np.abs(np.sqrt(hist[:ko + 1]) - np.sqrt(ho))) / np.sqrt(ho[0])
            assert rerr <= SPREAD_FACTOR * rs + 8 * eps, f"|r| err {rerr:.3g} vs oracle spread {rs:.3g}"
        else:
            assert np.array_equal(x, ref[0]), f"{variant}/{policy} x differs from hostloop"
            assert np.array_equal(hist[:ko + 1], ref[1][:ko + 1]), f"{variant}/{policy} history differs"
    h.close()


@pytest.mark.parametrize("dtype", DT)
def test_cg_converges_to_tolerance_like_the_oracle(dtype):
    _need_gpu()
    ro, ci, va = sp.poisson2d(24)
    n = len(ro) - 1
    b = sp.rhs(n, dtype=dtype)
    tol = 1e-8 if dtype == np.float64 else 1e-3
    xo, ho, ko = oracle.cg(ro, ci, va, b, kmax=2000, tol=tol)
    h = _cg(ro, ci, va, dtype)
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, b, 2000, tol, variant, policy)
        k = int(info[0])
        assert info[1] == 0 and abs(k - ko) <= 2 and hist[k] <= tol * tol
        assert np.all(np.isnan(hist[k + 1:]))
        a_x = oracle.csr_spmv(ro, ci, va, x.astype(np.float64).astype(dtype))
        res = b.astype(np.float64) - a_x.astype(np.float64)
        assert np.sqrt(res @ res) <= 50 * tol * (1 if dtype == np.float64 else 10)
    h.close()


@pytest.mark.parametrize("dtype", DT)
def test_cg_edge_cases(dtype):
    _need_gpu()
    from paper_2204_02064_b200 import CG
    # b = 0: no iteration, x = 0 (RC2)
    ro, ci, va = sp.poisson2d(9)
    h = _cg(ro, ci, va, dtype)
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, np.zeros(81, dtype=dtype), 10, 0.0, variant, policy)
        assert info.tolist() == [0, 0] and np.all(x == 0) and hist[0] == 0
        # k_max = 0: x = 0, history[0] = <b,b>
        b = sp.rhs(81, dtype=dtype)
        x, hist, info = _gpu_solve(h, b, 0, 0.0, variant, policy)
        assert info.tolist() == [0, 0] and np.all(x == 0)
        h0 = oracle.cg(ro, ci, va, b, kmax=0)[1][0]   # <b,b>: any order within 2 n u sum b^2
        assert abs(hist[0] - h0) <= 2 * 81 * 2.0 ** -53 * h0
    h.close()
    # A = 4 I: one exact step, then <r,r> = 0 stops the loop
    n = 5000
    h = CG(np.arange(n + 1), np.arange(n, dtype=np.int32), np.full(n, 4.0),
           dtype="f64" if dtype == np.float64 else "f32")
    b = sp.rhs(n, dtype=dtype)
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, b, 10, 0.0, variant, policy)
        assert info.tolist() == [1, 0] and np.array_equal(x, (b / dtype(4)).astype(dtype)) and hist[1] == 0
    h.close()
    # A = -I: breakdown at the first step (RC4)
    h = CG(np.arange(n + 1), np.arange(n, dtype=np.int32), np.full(n, -1.0),
           dtype="f64" if dtype == np.float64 else "f32")
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, b, 10, 0.0, variant, policy)
        assert info.tolist() == [0, 1]
    h.close()
    # 2x2 hand case
    h = CG(np.array([0, 2, 4]), np.array([0, 1, 0, 1], np.int32), np.array([4.0, 1, 1, 3]),
           dtype="f64" if dtype == np.float64 else "f32")
    x, hist, info = _gpu_solve(h, np.array([1.0, 2.0], dtype=dtype), 50, 1e-12 if dtype == np.float64 else 1e-6)
    assert info[0] <= 2 and np.allclose(x, [1 / 11, 7 / 11], atol=1e-12 if dtype == np.float64 else 1e-6)
    h.close()


def test_cg_solve_host_matches_device_path():
    _need_gpu()
    ro, ci, va = sp.poisson3d(12)
    n = len(ro) - 1
    b = sp.rhs(n)
    h = _cg(ro, ci, va, np.float64)
    x_d, hist_d, info_d = _gpu_solve(h, b, 30)
    x_h, hist_h, k, st = h.solve_host(b, 30)
    assert np.array_equal(x_d, x_h) and k == info_d[0] and st == 0
    assert np.array_equal(hist_d[:k + 1], hist_h[:k + 1])
    h.close()


def test_cg_rejects_bad_arguments():
    _need_gpu()
    from paper_2204_02064_b200 import CG
    from paper_2204_02064_b200._lib import PerksError
    with pytest.raises(PerksError):
        CG(np.array([0, 1]), np.array([5], np.int32), np.array([1.0]))   # column out of range
    with pytest.raises(PerksError):
        CG(np.array([0, 2, 1, 2]), np.array([0, 1], np.int32), np.array([1.0, 1.0]))
    h = CG(*sp.poisson2d(4))
    with pytest.raises(ValueError):
        h.solve(torch.zeros(16, dtype=torch.float32, device="cuda"), 3)
    h.close()


@pytest.mark.parametrize("wl", ["G2", "G3", "G4", "G5"])
def test_cg_fullsize_workloads(wl):
    """BASELINE-class sizes (DESIGN.md CG workloads), 12 iterations: oracle parity and
    bit-identity of the variants and policies at the size bench.py times."""
    _need_gpu()
    kind, size, dtype, _, _ = sp.CG_WORKLOADS[wl]
    ro, ci, va = sp.matrix(kind, size)
    n = len(ro) - 1
    b = sp.rhs(n, dtype=dtype)
    K = 12
    xo, ho, ko = oracle.cg(ro, ci, va, b, kmax=K, nthreads=oracle.max_threads())
    h = _cg(ro, ci, va, dtype)
    ref = None
    for variant, policy in POLICIES:
        x, hist, info = _gpu_solve(h, b, K, 0.0, variant, policy)
        assert info.tolist() == [K, 0]
        if ref is None:
            ref = x
            err = np.max(np.abs(x - xo)) / np.max(np.abs(xo))
            assert err <= XTOL[dtype], f"x rel err {err}"
            assert np.allclose(hist, ho, rtol=RTOL_HIST[dtype], atol=0)
        else:
            assert np.array_equal(x, ref), f"{variant}/{policy}"
    h.close()
