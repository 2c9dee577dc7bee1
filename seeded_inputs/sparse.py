"""Seeded synthetic sparse SPD matrices and right-hand sides for the CG workload (NEXT-3).

Input generation only: this module builds CSR arrays and vectors, and holds none of the
method's arithmetic (no SpMV, no inner products, no CG step).  Both the oracle side (tests)
and the CUDA side (tests, bench) draw their inputs from here.

The paper's CG datasets are SuiteSparse SPD matrices (Table V: 1,440 to
1,004,000 rows, 41,906 to 17,550,675 nonzeros), which are not available offline.  The
synthetic stand-ins keep their structure classes:

* ``poisson2d(nx, ny)``  — 5-point finite-difference Laplacian, Dirichlet (diag 4, off -1);
  the 2D-PDE class (fv1, shallow_water2, ecology2);
* ``poisson3d(n)``       — 7-point Laplacian (diag 6, off -1);
* ``box27(n)``           — 27-point 3D operator 27 I - B (B = the 3x3x3 all-ones box):
  SPD (eigenvalues 27 - prod(1 + 2 cos t_a) > 0), 27 nonzeros per interior row; the 3D FEM
  class of the large datasets (hood, BenElechi1, af_1_k101: 35-60 nonzeros per row);
* ``irregular(n, ...)``  — random symmetric pattern with a ragged, heavy-tailed degree
  distribution (a few rows hundreds of entries long) made strictly diagonally dominant,
  hence SPD: the load-imbalance class merge-based SpMV exists for.

Every row lists its columns strictly increasing; every diagonal entry is stored.  Values of
the structured operators are small integers (exact in any dtype); ``irregular`` uses dyadic
off-diagonals -m/64, m in 1..64, so every sum of them is exact too.
"""
from __future__ import annotations

import numpy as np

from . import SEED, field, splitmix64


def _finish(rows: np.ndarray, cols: np.ndarray, vals: np.ndarray, n: int):
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_off[1:])
    return row_off, cols.astype(np.int32), vals.astype(np.float64)


def _grid_operator(shape, offsets, weight_of):
    """CSR of sum_d weight_of(d) u(c + d) on a Dirichlet grid (C order, x fastest)."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    coords = np.indices(shape).reshape(len(shape), -1)
    idx = np.arange(n, dtype=np.int64)
    rows, cols, vals = [], [], []
    for d in offsets:
        q = coords + np.asarray(d, dtype=np.int64)[:, None]
        ok = np.all((q >= 0) & (q < np.asarray(shape)[:, None]), axis=0)
        lin = np.ravel_multi_index(tuple(q[:, ok]), shape)
        rows.append(idx[ok])
        cols.append(lin)
        vals.append(np.full(lin.shape[0], weight_of(d), dtype=np.float64))
    return _finish(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), n)


def poisson2d(nx: int, ny: int | None = None):
    """5-point Laplacian on an ny x nx grid: (row_off int64[n+1], col int32[nnz], val f64[nnz])."""
    ny = nx if ny is None else ny
    offs = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    return _grid_operator((ny, nx), offs, lambda d: 4.0 if d == (0, 0) else -1.0)


def poisson3d(n: int):
    """7-point Laplacian on an n^3 grid."""
    offs = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    return _grid_operator((n, n, n), offs, lambda d: 6.0 if d == (0, 0, 0) else -1.0)


def box27(n: int):
    """27 I - B on an n^3 grid (B = 3x3x3 all-ones box, Dirichlet): diag 26, off -1."""
    offs = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    return _grid_operator((n, n, n), offs, lambda d: 26.0 if d == (0, 0, 0) else -1.0)


def irregular(n: int, mean_degree: int = 12, seed: int = SEED, heavy_rows: int = 8,
              heavy_degree: int = 400):
    """Random symmetric SPD matrix with a ragged degree distribution.

    Off-diagonal pattern: each row i draws d_i partners, d_i geometric with the given mean
    (so many rows have 1-3 entries and some dozens), plus ``heavy_rows`` rows with
    ``heavy_degree`` partners; the pattern is symmetrised and deduplicated.  Off-diagonal
    values -m/64 (m = 1..64, from a counter-based hash of the unordered pair, so the
    matrix is symmetric); diagonal = sum |off-diagonal| + 1 (strict dominance => SPD)."""
    rng = np.random.default_rng(seed ^ 0x5D)
    deg = rng.geometric(1.0 / max(1, mean_degree // 2), size=n)
    heavy = rng.choice(n, size=min(heavy_rows, n), replace=False)
    deg[heavy] = heavy_degree
    deg = np.minimum(deg, n - 1)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = rng.integers(0, n, size=src.shape[0], dtype=np.int64)
    keep = src != dst
    a, b = np.minimum(src[keep], dst[keep]), np.maximum(src[keep], dst[keep])
    key = np.unique(a * n + b)
    a, b = key // n, key % n
    h = splitmix64((key.astype(np.uint64) ^ np.uint64(seed)))
    w = -((h >> np.uint64(58)).astype(np.float64) + 1.0) / 64.0          # -m/64, m in 1..64
    rows = np.concatenate([a, b])
    cols = np.concatenate([b, a])
    vals = np.concatenate([w, w])
    diag = np.bincount(rows, weights=-vals, minlength=n) + 1.0
    rows = np.concatenate([rows, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([cols, np.arange(n, dtype=np.int64)])
    vals = np.concatenate([vals, diag])
    return _finish(rows, cols, vals, n)


def rhs(n: int, dtype=np.float64, seed: int = SEED ^ 0xB):
    """Right-hand side b: counter-based values in [1, 2) (the stencil field recipe)."""
    return field((n,), dtype=dtype, seed=seed)


def matrix(kind: str, size: int):
    return {"poisson2d": lambda s: poisson2d(s), "poisson3d": poisson3d, "box27": box27,
            "irregular": lambda s: irregular(s)}[kind](size)


# CG workloads (CG rows): the Table V size classes on B200.
# name: (kind, size, dtype, iterations, description)
CG_WORKLOADS = {
    "G1": ("poisson2d", 64, np.float64, 100, "2D 5-point Poisson 64^2 fp64 (4,096 rows; oracle in seconds)"),
    "G2": ("poisson2d", 256, np.float64, 10000,
           "2D 5-point Poisson 256^2 fp64 (65,536 rows, 326,656 nnz; Table V D6-D7 class, fits on chip)"),
    "G3": ("poisson3d", 64, np.float64, 10000,
           "3D 7-point Poisson 64^3 fp64 (262,144 rows, 1.8M nnz; D11-D13 class, fits on chip)"),
    "G4": ("box27", 80, np.float64, 2000,
           "3D 27-point 80^3 fp64 (512,000 rows, 13.5M nnz, 166 MB CSR; D15-D20 class, exceeds L2)"),
    "G5": ("irregular", 200000, np.float64, 2000,
           "irregular SPD, 200,000 rows, ragged degrees (merge-path load-balance case)"),
}
