"""PERKS performance model (§4) and concurrency counts.

Analysis layer only (offline, not called by the kernels).  bench.py uses it to
report the projected peak ℙ and ℳ/ℙ next to the measured ℳ; tests pin every
formula to the paper's printed worked examples (tests/golden/paper_model.json).

Units: following the paper's worked examples, D and D_cache are counted in
ELEMENTS (cells) and multiplied by the element size 𝔖 inside the time formulas
(P:562 Eq. time_gm: T_gm = A_gm·𝔖/B_gm).
"""
from __future__ import annotations

from dataclasses import dataclass


def A_gm(D: float, D_cache: float, N: int) -> float:
    """Eq.: A_gm(D) = 2·N·D_uncache + 2·D_cache (elements)."""
    return 2.0 * N * (D - D_cache) + 2.0 * D_cache


def T_gm(D: float, D_cache: float, N: int, S: int, B_gm: float) -> float:
    """Eq. time_gm: T_gm = A_gm·𝔖 / B_gm (seconds)."""
    return A_gm(D, D_cache, N) * S / B_gm


def A_sm(D_sm_cache: float, N: int) -> float:
    """Eq.: A_sm = 2·(N-1)·D^sm_cache (elements)."""
    return 2.0 * (N - 1) * D_sm_cache


def T_sm(D_sm_cache: float, N: int, S: int, B_sm: float, A_sm_kernel: float = 0.0) -> float:
    """Eq. time_sm: T_sm = (A_sm(D^sm_cache) + A_sm(KERNEL))·𝔖 / B_sm."""
    return (A_sm(D_sm_cache, N) + A_sm_kernel) * S / B_sm


def T_halo(A_halo: float, S: int, B_gm: float) -> float:
    """Eq. perkhalo: T_gm(H(D_cache)) = A(H(D_cache))·𝔖 / B_gm."""
    return A_halo * S / B_gm


def T_perks(t_gm: float, t_halo: float, t_sm: float) -> float:
    """Eq. maxlat: T_PERKS = max(T_gm + T_halo, T_sm)."""
    return max(t_gm + t_halo, t_sm)


def P_peak(D: float, N: int, t_perks: float) -> float:
    """Eq. maxpeak: ℙ = D·N / T_PERKS (cells per second)."""
    return D * N / t_perks


def halo_elements_2d(N: int, n_tb: int, tile_x: int, tile_y: int, rad: int = 1) -> float:
    """Halo accesses of the §4.2 example: N·2·TBs·(tile_y·2 + tile_x·2)·rad.

    The paper's 216·(136·2+256·2) counts, per TB and step, the two vertical edges
    (136 cells) and two horizontal edges (256 cells) of its 256×136 cached tile,
    times 2 (one store + one load).
    """
    return float(N) * 2 * n_tb * (tile_y * 2 + tile_x * 2) * rad


def table3_gm_ops(tb_per_smx: int, tile_x: int = 256, tile_y: int = 8, rad: int = 1):
    """Table III static concurrency: GM load and store ops per SMX.

    Loads per TB = (tile_x+2r)·(tile_y+2r) (tile plus halo incl. corners),
    stores per TB = tile_x·tile_y.
    """
    loads = (tile_x + 2 * rad) * (tile_y + 2 * rad) * tb_per_smx
    stores = tile_x * tile_y * tb_per_smx
    return loads, stores


def b_sm(n_sm: int, bytes_per_clk: int, clk_hz: float) -> float:
    """Aggregate shared-memory bandwidth: SMs × bytes/clk × clock."""
    return n_sm * bytes_per_clk * clk_hz


@dataclass
class Projection:
    t_gm: float
    t_halo: float
    t_sm: float
    t_perks: float
    peak_cells_per_s: float


def project(D, D_cache, N, S, B_gm, A_halo=0.0, D_sm_cache=0.0, B_sm=float("inf"),
            A_sm_kernel=0.0, A_gm_elems=None) -> Projection:
    """ℙ for one configuration (Eqs. basic…maxpeak).  ``A_gm_elems`` replaces Eq. when a
    kernel's global traffic is not of the cached-fraction form (two steps per pass: N·D)."""
    tg = T_gm(D, D_cache, N, S, B_gm) if A_gm_elems is None else A_gm_elems * S / B_gm
    th = T_halo(A_halo, S, B_gm)
    ts = T_sm(D_sm_cache, N, S, B_sm, A_sm_kernel) if B_sm != float("inf") else 0.0
    tp = T_perks(tg, th, ts)
    return Projection(tg, th, ts, tp, P_peak(D, N, tp))


def little_concurrency(throughput_per_cycle: float, latency_cycles: float) -> float:
    """C_hw = THR·L (Little's law)."""
    return throughput_per_cycle * latency_cycles


def efficiency(c_sw: float, c_hw: float) -> float:
    """𝔈(C_sw, C_hw) = min(1, C_sw/C_hw) (100% iff C_sw ≥ C_hw)."""
    return 1.0 if c_sw >= c_hw else c_sw / c_hw
