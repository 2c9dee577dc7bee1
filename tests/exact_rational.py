"""Independent exact-rational stencil evaluator (pure Python ``fractions``).

Used only to PIN the oracle: it shares nothing with ``oracle/`` (no numpy, no
C, no fma) and evaluates the definition x^{k+1}(c) = sum_p w_p x^k(c+d_p)
 exactly, with FRAME or PERIODIC boundaries, on tiny grids.
Inside the "exactness window" every intermediate value is representable in the
dtype, so a correct dtype implementation must match it bit for bit regardless
of summation order.
"""
from fractions import Fraction


def run_exact(u0, dims, offsets, weights, steps, periodic=False):
    """u0: flat list of Fractions in C order; dims=(nx, ny, nz)."""
    nx, ny, nz = dims
    ndim = 3 if nz > 1 else 2
    r = max(max(abs(d) for d in off) for off in offsets)
    w = [Fraction(x) for x in weights]
    cur = list(u0)
    for _ in range(steps):
        nxt = list(cur)
        for z in range(nz):
            for y in range(ny):
                for x in range(nx):
                    if not periodic:
                        if x < r or x >= nx - r or y < r or y >= ny - r:
                            continue
                        if ndim == 3 and (z < r or z >= nz - r):
                            continue
                    s = Fraction(0)
                    for (dx, dy, dz), wp in zip(offsets, w):
                        qx, qy, qz = x + dx, y + dy, z + dz
                        if periodic:
                            qx %= nx
                            qy %= ny
                            qz %= nz
                        s += wp * cur[(qz * ny + qy) * nx + qx]
                    nxt[(z * ny + y) * nx + x] = s
        cur = nxt
    return cur
