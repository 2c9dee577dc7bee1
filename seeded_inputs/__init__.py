"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only produces initial
fields and coefficient lists.  Both ``oracle/`` (via the tests) and the product
benchmarks draw their inputs from here, so the two paths see identical bytes.

Field recipe (SURVEY §8(c) reading 13): the paper's
StencilGen data is unavailable, so every cell gets a counter-based
value ``u0[i] = 1 + m(i) * 2^-p`` where ``m(i)`` is the top ``p`` bits of
``splitmix64(seed XOR i)`` and ``i`` the GLOBAL C-order linear index
(z*ny*nx + y*nx + x).  ``p`` = 52 (f64) / 23 (f32) gives exactly representable
values in [1, 2); ``p`` = 10 gives 10-bit dyadic values for exact-rational tests.
Because the generator is counter based, each rank of a slab decomposition can
produce its own slab (``z_offset``) and the concatenation equals the global field.

Coefficient presets (reading 2): dyadic, convex, summing to exactly 1, listed in
the canonical accumulation order (reading 5):
  * 2d5pt   W,E,S,C,N             C=1/2, others 1/8          (Fig. 6 order)
  * 2d9pt   3x3 box, (dy,dx) lexicographic, w=(2-|dx|)(2-|dy|)/16
  * 3d7pt   W,E,S,C,N,B,F         C=1/4, others 1/8
  * 3d27pt  3x3x3 box, (dz,dy,dx) lexicographic, w=prod(2-|d|)/64
"""
from __future__ import annotations

import numpy as np

SEED = 0x220402064
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser on uint64 (wrapping arithmetic)."""
    z = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += _GOLDEN
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def _bits_for(dtype, bits):
    if bits is not None:
        return bits
    return 52 if np.dtype(dtype) == np.float64 else 23


def field(shape, dtype=np.float64, seed: int = SEED, bits: int | None = None,
          index_offset: int = 0) -> np.ndarray:
    """Field of ``shape`` (C order) with values 1 + m*2^-bits in [1,2)."""
    dtype = np.dtype(dtype)
    p = _bits_for(dtype, bits)
    n = int(np.prod(shape))
    out = np.empty(n, dtype=dtype)
    chunk = 1 << 24
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = np.arange(s + index_offset, e + index_offset, dtype=np.uint64)
        z = splitmix64(idx ^ np.uint64(seed))
        m = (z >> np.uint64(64 - p)).astype(np.float64)
        out[s:e] = (1.0 + m * 2.0 ** (-p)).astype(dtype)
    return out.reshape(shape)


def field_torch(shape, dtype, device, seed: int = SEED, bits: int | None = None,
                index_offset: int = 0):
    """Same values as :func:`field`, generated with torch int64 ops on ``device``.

    int64 arithmetic wraps like uint64; logical right shifts are emulated with a
    mask, so the bit pattern equals the numpy uint64 version exactly.
    """
    import torch

    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}[np.dtype(dtype)]
    p = _bits_for(dtype, bits)
    n = 1
    for s_ in shape:
        n *= int(s_)

    def c64(v):  # uint64 constant -> int64 with the same bits
        v = int(v) & 0xFFFFFFFFFFFFFFFF
        return v - (1 << 64) if v >= (1 << 63) else v

    def lsr(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)

    out = torch.empty(n, dtype=tdt, device=device)
    chunk = 1 << 26
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        z = torch.arange(s + index_offset, e + index_offset, dtype=torch.int64, device=device)
        z = z ^ c64(seed)
        z = z + c64(_GOLDEN)
        z = (z ^ lsr(z, 30)) * c64(_M1)
        z = (z ^ lsr(z, 27)) * c64(_M2)
        z = z ^ lsr(z, 31)
        m = lsr(z, 64 - p).to(torch.float64)
        out[s:e] = (1.0 + m * 2.0 ** (-p)).to(tdt)
    return out.reshape(tuple(int(s_) for s_ in shape))


# ---------------------------------------------------------------- presets

def preset(name: str):
    """Return (offsets [(dx,dy,dz)...], weights [float]) in canonical order."""
    if name == "2d5pt":
        offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 0, 0), (0, 1, 0)]   # W,E,S,C,N
        w = [1 / 8, 1 / 8, 1 / 8, 1 / 2, 1 / 8]
    elif name == "2d9pt":
        offs, w = [], []
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                offs.append((dx, dy, 0))
                w.append((2 - abs(dx)) * (2 - abs(dy)) / 16)
    elif name == "3d7pt":
        offs = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 0, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
        w = [1 / 8, 1 / 8, 1 / 8, 1 / 4, 1 / 8, 1 / 8, 1 / 8]                # W,E,S,C,N,B,F
    elif name == "3d27pt":
        offs, w = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    offs.append((dx, dy, dz))
                    w.append((2 - abs(dx)) * (2 - abs(dy)) * (2 - abs(dz)) / 64)
    elif name == "3d19pt":
        # Table II "poisson(1,38)": 19 points = the 3x3x3 cube without its 8 corners (reading
        # R3b); dyadic convex weights C=1/4, faces 1/16, edges 1/32 (sum exactly 1)
        offs, w = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    m = abs(dx) + abs(dy) + abs(dz)
                    if m == 3:
                        continue
                    offs.append((dx, dy, dz))
                    w.append({0: 1 / 4, 1: 1 / 16, 2: 1 / 32}[m])
    elif name == "3d13pt":
        # Table II 3d13pt(2,26): the radius-2 3D star, (dz,dy,dx) lexicographic; dyadic convex
        # weights: centre 1/16, distance 1 1/8, distance 2 1/32 (sum exactly 1)
        offs, w = [], []
        for dz in range(-2, 3):
            for dy in range(-2, 3):
                for dx in range(-2, 3):
                    if (dx != 0) + (dy != 0) + (dz != 0) > 1:
                        continue
                    k = abs(dx) + abs(dy) + abs(dz)
                    offs.append((dx, dy, dz))
                    w.append({0: 1 / 16, 1: 1 / 8, 2: 1 / 32}[k])
    elif name == "3d17pt":
        # Table II 3d17pt(1,34): order 1, 17 points.  The text fixes only (order, FLOPs); no
        # 17-point subset of the 3x3x3 cube is invariant under all cube symmetries (orbits 1, 6, 12,
        # 8), so reading R3e takes the set invariant under the symmetries that keep z:
        # the centre plane's 3x3 box (9) plus the 8 cube corners (|dx| = |dy| = |dz| = 1).
        # (dz,dy,dx) lexicographic; dyadic convex weights: centre 1/4, in-plane faces 1/8, in-plane
        # corners 1/32, cube corners 1/64 (sum exactly 1)
        offs, w = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if dz != 0 and (dx == 0 or dy == 0):
                        continue
                    offs.append((dx, dy, dz))
                    m = abs(dx) + abs(dy)
                    w.append(1 / 64 if dz != 0 else {0: 1 / 4, 1: 1 / 8, 2: 1 / 32}[m])
    elif name in STAR_RADIUS:
        # Table II high-order stars 2ds9pt / 2d13pt / 2d17pt / 2d21pt / 2ds25pt (radius 2..6):
        # the 4r+1 points (0,dy) and (dx,0), (dy,dx) lexicographic; dyadic convex weights: centre
        # 2^-r, distance k along each arm 2^-(k+2) (sum exactly 1)
        r = STAR_RADIUS[name]
        offs, w = [], []
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                if dx != 0 and dy != 0:
                    continue
                k = abs(dx) + abs(dy)
                offs.append((dx, dy, 0))
                w.append(2.0 ** -r if k == 0 else 2.0 ** -(k + 2))
    elif name == "2d25pt":
        # Table II 2d25pt: the 5x5 box (radius 2), (dy,dx) lexicographic; binomial weights
        # (1,4,6,4,1)/16 per axis (dyadic, sum exactly 1)
        b = {-2: 1, -1: 4, 0: 6, 1: 4, 2: 1}
        offs, w = [], []
        for dy in range(-2, 3):
            for dx in range(-2, 3):
                offs.append((dx, dy, 0))
                w.append(b[dx] * b[dy] / 256)
    else:
        raise KeyError(name)
    return offs, w


STAR_RADIUS = {"2ds9pt": 2, "2d13pt": 3, "2d17pt": 4, "2d21pt": 5, "2ds25pt": 6}
PRESET_NDIM = {"2d5pt": 2, "2d9pt": 2, "3d7pt": 3, "3d27pt": 3, "3d19pt": 3, "2d25pt": 2, "3d13pt": 3, "3d17pt": 3,
               **{k: 2 for k in STAR_RADIUS}}


def random_convex_weights(npts: int, dtype=np.float64, seed: int = 7) -> list[float]:
    """Random positive weights (seeded), normalised to sum ~1, then dtype-rounded."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.5, 1.5, size=npts)
    w = w / w.sum()
    return [float(v) for v in w.astype(dtype)]


# ---------------------------------------------------------------- configs

# BASELINE.json configs; C5 is per-GPU slab, global z = 1024*N.
CONFIGS = {
    "C1": dict(stencil="2d5pt", dtype="f64", shape=(128, 128), steps=100),
    "C2": dict(stencil="2d9pt", dtype="f32", shape=(3072, 3072), steps=1000),
    "C3": dict(stencil="3d7pt", dtype="f64", shape=(256, 256, 256), steps=1000),
    "C4": dict(stencil="3d27pt", dtype="f32", shape=(512, 512, 512), steps=500),
    "C5": dict(stencil="3d7pt", dtype="f64", shape=(1024, 1024, 1024), steps=100),
}
# Cached-fraction sweep points (not BASELINE configs): 3D domains from fully
# on-chip-cacheable to C3's size, the 3D analogue of the paper's small/large domains (Fig. 5).
SWEEP_CONFIGS = {
    "S3_128": dict(stencil="3d7pt", dtype="f64", shape=(128, 128, 128), steps=1000),
    "S3_160": dict(stencil="3d7pt", dtype="f64", shape=(160, 160, 160), steps=1000),
    "S3_192": dict(stencil="3d7pt", dtype="f64", shape=(192, 192, 192), steps=1000),
    "S3_224": dict(stencil="3d7pt", dtype="f64", shape=(224, 224, 224), steps=1000),
    "S27_256": dict(stencil="3d27pt", dtype="f32", shape=(256, 256, 256), steps=500),
    # 2D domain sweep (C2's stencil): from one cluster to the full on-chip capacity
    "S2_256": dict(stencil="2d9pt", dtype="f32", shape=(256, 256), steps=1000),
    "S2_512": dict(stencil="2d9pt", dtype="f32", shape=(512, 512), steps=1000),
    "S2_1024": dict(stencil="2d9pt", dtype="f32", shape=(1024, 1024), steps=1000),
    "S2_2048": dict(stencil="2d9pt", dtype="f32", shape=(2048, 2048), steps=1000),
    "S2_2560": dict(stencil="2d9pt", dtype="f32", shape=(2560, 2560), steps=1000),
    "S2d_1024": dict(stencil="2d5pt", dtype="f64", shape=(1024, 1024), steps=1000),
    "S2d_1536": dict(stencil="2d5pt", dtype="f64", shape=(1536, 1536), steps=1000),
    # Table II high-order stencils on the general kernels (k2d_wide.cu), fully cacheable size
    "W_2ds9pt": dict(stencil="2ds9pt", dtype="f32", shape=(1536, 1536), steps=1000),
    "W_2d13pt": dict(stencil="2d13pt", dtype="f32", shape=(1536, 1536), steps=1000),
    "W_2ds25pt": dict(stencil="2ds25pt", dtype="f32", shape=(1536, 1536), steps=1000),
    "W_2d25pt": dict(stencil="2d25pt", dtype="f32", shape=(1536, 1536), steps=1000),
    "W_2ds9pt_f64": dict(stencil="2ds9pt", dtype="f64", shape=(1536, 768), steps=1000),
}
