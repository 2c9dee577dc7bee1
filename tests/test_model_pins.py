"""Pins for the PERKS performance model (paper_2204_02064_b200/model.py) against
the values the paper prints (tests/golden/paper_model.json, each entry cited)."""
import json
import os

import pytest

from paper_2204_02064_b200 import model

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_model.json")))


def test_large_domain_worked_example():
    g = GOLD["large_domain_example"]
    t_gm = model.T_gm(g["D"], g["D_cache"], g["N"], g["S"], g["B_gm"])
    assert round(t_gm * 1e6, 2) == g["T_gm_us"]
    a_halo = model.halo_elements_2d(g["N"], g["n_tb"], g["tile_x"], g["tile_y"])
    t_h = model.T_halo(a_halo, g["S"], g["B_gm"])
    assert round(t_h * 1e6, 2) == g["T_halo_us"]
    p = model.project(g["D"], g["D_cache"], g["N"], g["S"], g["B_gm"], A_halo=a_halo)
    assert round(p.peak_cells_per_s / 1e9, 2) == g["P_gcells"]
    assert round(100 * g["measured_gcells"] / (p.peak_cells_per_s / 1e9), 2) == g["measured_frac_pct"]
    # the cached region is 216 TBs of 256x136 cells = 3072x2448 (P:609 geometry)
    assert g["n_tb"] * g["tile_x"] * g["tile_y"] == g["D_cache"]


def test_small_domain_worked_example():
    g = GOLD["small_domain_example"]
    bsm = model.b_sm(g["n_sm"], g["bytes_per_clk"], g["clk_hz"])
    assert abs(bsm / 1e12 - 19.5) < 0.05  # [draft] P:495 quotes 19.5 TB/s
    a_k = g["D"] * g["N"] * 4
    t_sm = model.T_sm(g["D_sm_cache"], g["N"], g["S"], bsm, A_sm_kernel=a_k)
    assert round(t_sm * 1e3, 1) == g["T_sm_ms"]
    # fully cached: T_gm counts only the one-time 2*D_cache term
    p = model.project(g["D"], g["D"], g["N"], g["S"], 1555e9, D_sm_cache=g["D_sm_cache"],
                      B_sm=bsm, A_sm_kernel=a_k)
    assert p.t_perks == pytest.approx(t_sm)
    assert round(p.peak_cells_per_s / 1e9, 2) == g["P_gcells"]
    assert round(100 * g["measured_gcells"] / (p.peak_cells_per_s / 1e9), 2) == g["measured_frac_pct"]


def test_table3_counts():
    for tb, loads, stores in GOLD["table3"]["rows"]:
        assert model.table3_gm_ops(tb) == (loads, stores)


def test_agm_limits():
    # no caching -> 2·N·D ; full caching -> 2·D (one load + one store in total)
    assert model.A_gm(100, 0, 7) == 1400
    assert model.A_gm(100, 100, 7) == 200
    assert model.efficiency(5, 10) == 0.5 and model.efficiency(20, 10) == 1.0


def test_table2_flops_of_presets():
    """Reading R3: flops/cell = 2·|P| (FMA counted as 2) matches Table II for the hot-path shapes."""
    import seeded_inputs as si
    rows = {r[0]: (r[1], r[2]) for r in GOLD["table2"]["rows"]}
    for name in ("2d5pt", "2d9pt", "3d7pt", "3d27pt", "3d17pt", "3d13pt", "2ds9pt", "2d13pt",
                 "2d17pt", "2d21pt", "2d25pt"):
        offs, _ = si.preset(name)
        order = max(max(abs(d) for d in o) for o in offs)
        assert (order, 2 * len(offs)) == rows[name], name
    offs, _ = si.preset("3d19pt")  # Table II "poisson" (reading R3b)
    assert (max(max(abs(d) for d in o) for o in offs), 2 * len(offs)) == rows["poisson"]
