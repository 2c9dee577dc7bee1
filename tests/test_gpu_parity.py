"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): max relative error <= 1e-12 (fp64) / 1e-5 (fp32) after T steps,
frame (boundary) cells bit-exact.  The design (reading R5: canonical FMA order, one rounding per
term) makes every cell bit-exact, which these tests also assert.  Outputs and workspaces are
NaN-poisoned before each run so an unwritten cell cannot pass.
"""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.float64: 1e-12, np.float32: 1e-5}
VARIANTS = ["hostloop", "persistent", "perks"]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run_gpu(u0, name, w, steps, variant):
    from paper_2204_02064_b200 import Stencil
    offs, _ = si.preset(name)
    st = Stencil(u0.shape, offs, w, dtype=u0.dtype)
    x = torch.from_numpy(u0).cuda()
    out = torch.full_like(x, float("nan"))
    ws = None
    if steps > 0:
        nb = st.workspace_bytes(variant)
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device="cuda")
        ws.view(torch.uint8).fill_(0xFF)  # NaN pattern for float buffers
    st.run(x, steps, variant, out=out, workspace=ws)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    st.close()
    return res


def _check(gpu, ref, u0, dtype, exact=True):
    assert not np.isnan(gpu).any(), "unwritten (NaN) cells"
    # frame cells bit-exact (reading R1)
    fr = np.ones(u0.shape, dtype=bool)
    fr[(slice(1, -1),) * u0.ndim] = False
    assert np.array_equal(gpu[fr], u0[fr])
    rel = np.max(np.abs(gpu.astype(np.float64) - ref) / np.abs(ref.astype(np.float64)))
    assert rel <= TOL[dtype], f"max rel err {rel}"
    if exact:
        nbad = int(np.sum(gpu != ref))
        assert nbad == 0, f"{nbad} cells differ from the oracle (max rel {rel})"


CASES_2D = [(3, 3), (5, 7), (17, 33), (67, 131), (128, 128), (130, 260), (257, 300), (500, 100)]
CASES_3D = [(3, 3, 3), (5, 6, 7), (9, 17, 33), (20, 35, 70), (34, 40, 132), (16, 40, 64), (37, 24, 128)]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("name", ["2d5pt", "2d9pt"])
@pytest.mark.parametrize("shape", CASES_2D)
def test_parity_2d(variant, dtype, name, shape):
    _need_gpu()
    u0 = si.field(shape, dtype=dtype, seed=101)
    offs, w = si.preset(name)
    for T in (1, 2, 7):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        gpu = _run_gpu(u0, name, w, T, variant)
        _check(gpu, ref, u0, dtype)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("name", ["3d7pt", "3d27pt", "3d19pt"])
@pytest.mark.parametrize("shape", CASES_3D)
def test_parity_3d(variant, dtype, name, shape):
    _need_gpu()
    u0 = si.field(shape, dtype=dtype, seed=202)
    offs, w = si.preset(name)
    for T in (1, 2, 5):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        try:
            gpu = _run_gpu(u0, name, w, T, variant)
        except Exception as e:  # PERKS 3D may not be planned for every domain
            if variant == "perks" and "UNSUPPORTED" in str(e):
                pytest.skip(str(e))
            raise
        _check(gpu, ref, u0, dtype)


@pytest.mark.parametrize("name,shape,dtype", [
    ("2d9pt", (300, 520), np.float32), ("2d5pt", (128, 128), np.float64),
    ("3d7pt", (24, 40, 64), np.float64), ("3d27pt", (20, 36, 128), np.float32),
    ("3d19pt", (22, 30, 72), np.float64), ("3d19pt", (18, 33, 136), np.float32)])
def test_random_weights_and_cross_variant(name, shape, dtype):
    """Non-symmetric random weights; all variants bit-identical to each other and the oracle."""
    _need_gpu()
    offs, _ = si.preset(name)
    w = si.random_convex_weights(len(offs), dtype, seed=5)
    u0 = si.field(shape, dtype=dtype, seed=303)
    T = 9
    ref = oracle.run(u0, offs, w, T, nthreads=4)
    outs = {}
    for v in VARIANTS:
        try:
            outs[v] = _run_gpu(u0, name, w, T, v)
        except Exception as e:
            if v == "perks" and "UNSUPPORTED" in str(e):
                continue
            raise
        _check(outs[v], ref, u0, dtype)
    vs = list(outs)
    for a in vs[1:]:
        assert np.array_equal(outs[vs[0]], outs[a])


@pytest.mark.parametrize("variant", VARIANTS + ["auto"])
def test_steps_zero_copies_input(variant):
    _need_gpu()
    u0 = si.field((33, 65), dtype=np.float32)
    offs, w = si.preset("2d9pt")
    gpu = _run_gpu(u0, "2d9pt", w, 0, variant)
    assert np.array_equal(gpu, u0)


def test_composability_on_gpu():
    """run(T1) then run(T2) == run(T1+T2), bit-exact, for every variant."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset("2d9pt")
    u0 = si.field((200, 384), dtype=np.float32)
    st = Stencil(u0.shape, offs, w, dtype=np.float32)
    x = torch.from_numpy(u0).cuda()
    for v in VARIANTS:
        a = st.run(st.run(x, 3, v), 4, v)
        b = st.run(x, 7, v)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    st.close()


def test_errors_on_gpu():
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200._lib import PerksError
    offs, w = si.preset("2d5pt")
    st = Stencil((16, 16), offs, w, dtype="f64")
    x = torch.ones((16, 16), dtype=torch.float64, device="cuda")
    with pytest.raises(PerksError) as e:  # in-place is rejected (Jacobi)
        st.run(x, 1, "hostloop", out=x)
    assert e.value.name == "PERKS_ERR_ALIAS"
    with pytest.raises(PerksError) as e:  # too-small workspace
        st.run(x, 2, "hostloop", workspace=torch.empty(256, dtype=torch.uint8, device="cuda"))
    assert e.value.name == "PERKS_ERR_WORKSPACE"
    with pytest.raises(PerksError) as e:
        st.run(x, -1, "hostloop")
    assert e.value.name == "PERKS_ERR_INVALID_ARGUMENT"
    st.close()


def test_run_host_e2e():
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset("3d7pt")
    u0 = si.field((16, 24, 40), dtype=np.float64)
    st = Stencil(u0.shape, offs, w, dtype="f64")
    got = st.run_host(u0, 6, "auto")
    ref = oracle.run(u0, offs, w, 6)
    assert np.array_equal(got, ref)
    st.close()


@pytest.mark.parametrize("shape,dtype,name", [((128, 128), np.float64, "2d5pt"),
                                              ((500, 250), np.float32, "2d9pt"),
                                              ((9, 33), np.float64, "2d9pt")])
def test_small_domain_uses_cluster_kernel(shape, dtype, name):
    """Small 2D domains run in one thread-block cluster (registers + DSMEM halo, cluster barrier),
    bit-exact vs the oracle for a long run (T=100, the C1 step count)."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=dtype)
    q = st.query("perks")
    st.close()
    assert q["kernel"].startswith("perks2d_cluster"), q
    u0 = si.field(shape, dtype=dtype, seed=404)
    ref = oracle.run(u0, offs, w, 100, nthreads=4)
    _check(_run_gpu(u0, name, w, 100, "perks"), ref, u0, dtype)


@pytest.mark.parametrize("nsm", ["0", "1", "3", ""])
@pytest.mark.parametrize("zigzag", ["0", "1"])
@pytest.mark.parametrize("name,dtype", [("3d7pt", np.float64), ("3d27pt", np.float32)])
def test_perks3d_cache_and_zigzag(monkeypatch, nsm, zigzag, name, dtype):
    """PERKS-3D: cached planes (shared-memory slots spread through each CTA's segment, halo-ring
    refresh + perimeter publish) and zig-zag traversal are bit-exact for any cache size, both
    traversal directions and both step parities."""
    _need_gpu()
    monkeypatch.setenv("PERKS_P3D_CACHE", "1")
    if nsm:
        monkeypatch.setenv("PERKS_P3D_NSM", nsm)
    monkeypatch.setenv("PERKS_ZIGZAG", zigzag)
    shape = (45, 50, 64)
    u0 = si.field(shape, dtype=dtype, seed=606)
    offs, w = si.preset(name)
    for T in (5, 6):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


@pytest.mark.parametrize("shape,name", [((1000, 1500), "2d9pt"), ((517, 3072), "2d5pt"),
                                        ((449, 2049), "2d9pt")])
def test_strip_kernel(monkeypatch, shape, name):
    """Wide fp32 2D domains as full-width strips (opt-in, PERKS_STRIP=1: edge rows first, LL-tag
    exchange with the strips above/below only); bit-exact vs the oracle, ragged last strip."""
    _need_gpu()
    monkeypatch.setenv("PERKS_STRIP", "1")
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=np.float32)
    q = st.query("perks")
    st.close()
    assert q["kernel"].startswith("perks2d_strip"), q
    u0 = si.field(shape, dtype=np.float32, seed=707)
    for T in (1, 2, 7, 40):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, np.float32)


@pytest.mark.parametrize("nsm,ntm", [("0", ""), ("2", ""), ("0", "1"), ("3", "5")])
@pytest.mark.parametrize("wsg", ["0", "1", "2"])
@pytest.mark.parametrize("name,dtype,shape", [("3d7pt", np.float64, (70, 33, 72)),
                                              ("3d27pt", np.float32, (61, 40, 136))])
def test_perks3d_tmem_tier(monkeypatch, nsm, ntm, wsg, name, dtype, shape):
    """PERKS-3D Tensor-Memory cache tier (tmem.cuh): planes kept in TMEM across steps (tcgen05.st
    at write-back, tcgen05.ld + staging into the ring slot one arrival ahead), alone or mixed
    with the shared-memory tier, both warp-specialised geometries, long units (one z-chunk),
    ragged tiles in x and y, both step parities: bit-exact vs the oracle."""
    _need_gpu()
    monkeypatch.setenv("PERKS_P3D_CACHE", "1")
    monkeypatch.setenv("PERKS_P3D_NSM", nsm)
    if ntm:
        monkeypatch.setenv("PERKS_P3D_NTM", ntm)
    monkeypatch.setenv("PERKS_WSG", wsg)
    monkeypatch.setenv("PERKS_S3D_NZC", "1")
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=dtype)
    q = st.query("perks")
    st.close()
    assert q["cached_cells_tmem"] > 0 and q["tmem_cols_per_cta"] > 0, q
    u0 = si.field(shape, dtype=dtype, seed=808)
    for T in (1, 4, 7):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


# k2d_perks.cu configuration index -> tile (16-warp TMEM-row tiles first, then 8-warp tiles, then
# forced-only alternatives: three 8-warp tiles and, fp32, the one-warp-per-band V=8 tile)
TILE_CFGS = {np.float32: [(256, 256), (256, 192), (256, 128), (128, 128), (128, 64), (128, 32),
                          (256, 256), (256, 192), (256, 128), (256, 256)],
             np.float64: [(128, 128), (128, 96), (128, 64), (128, 32), (64, 16),
                          (128, 128), (128, 96), (128, 64)]}


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("name", ["2d5pt", "2d9pt"])
def test_perks2d_every_tile_config(monkeypatch, dtype, name):
    """Every PERKS-2D tile configuration (k2d_perks.cu, forced with PERKS_P2D_CFG) — registers,
    shared-memory and TMEM row tiers — on a domain of 2.5 x 1.5 tiles (ragged in x and y, several
    CTAs exchanging edges), bit-exact vs the oracle."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    for cfg, (tx, ty) in enumerate(TILE_CFGS[dtype]):
        monkeypatch.setenv("PERKS_P2D_CFG", str(cfg))
        shape = (ty + ty // 2 + 3, 2 * tx + tx // 2 + 4)  # (ny, nx)
        st = Stencil(shape, offs, w, dtype=dtype)
        q = st.query("perks")
        st.close()
        assert q["kernel"].startswith("perks2d_") and f"_t{tx}x{ty}" in q["kernel"], (cfg, q["kernel"])
        u0 = si.field(shape, dtype=dtype, seed=909 + cfg)
        for T in (1, 6):
            ref = oracle.run(u0, offs, w, T, nthreads=8)
            _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


WIDE_PRESETS = ["2ds9pt", "2d13pt", "2d17pt", "2d21pt", "2ds25pt", "2d25pt"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("name", WIDE_PRESETS)
@pytest.mark.parametrize("shape", [(13, 13), (67, 131), (150, 300), (300, 270)])
def test_parity_wide_2d(variant, dtype, name, shape):
    """Table II high-order stencils (radius 2..6) on the general 2D kernels (k2d_wide.cu): every
    variant bit-exact vs the oracle; domains from the minimum (2r+1 for r = 6) to several tiles
    with ragged edges (the PERKS tile exchange crosses tile corners for the 5x5 box)."""
    _need_gpu()
    offs, w = si.preset(name)
    r = max(max(abs(a), abs(b)) for a, b, _ in offs)
    if min(shape) < 2 * r + 1:
        pytest.skip("domain below 2r+1")
    u0 = si.field(shape, dtype=dtype, seed=1001)
    for T in (1, 5):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu_offs(u0, offs, w, T, variant), ref, u0, dtype)


def _run_gpu_offs(u0, offs, w, steps, variant):
    from paper_2204_02064_b200 import Stencil
    st = Stencil(u0.shape, offs, w, dtype=u0.dtype)
    x = torch.from_numpy(u0).cuda()
    out = torch.full_like(x, float("nan"))
    nb = st.workspace_bytes(variant)
    ws = torch.empty(max(nb, 256), dtype=torch.uint8, device="cuda")
    ws.fill_(0xFF)
    st.run(x, steps, variant, out=out, workspace=ws)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    st.close()
    return res


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_wide_2d_any_order_and_random_weights(dtype):
    """Point sets with no specialised kernel — a reversed 2d9pt list, an asymmetric radius-3 set —
    with random weights: all variants bit-identical to each other and to the oracle (the list order
    is the accumulation order, reading R5)."""
    _need_gpu()
    o9, _ = si.preset("2d9pt")
    asym = [(0, 0, 0), (3, 0, 0), (-1, 2, 0), (2, -3, 0), (-3, -1, 0), (1, 1, 0), (0, 3, 0)]
    for offs in (o9[::-1], asym):
        w = si.random_convex_weights(len(offs), dtype, seed=17)
        u0 = si.field((140, 290), dtype=dtype, seed=1002)
        ref = oracle.run(u0, offs, w, 6, nthreads=8)
        outs = [_run_gpu_offs(u0, offs, w, 6, v) for v in VARIANTS]
        for o in outs:
            _check(o, ref, u0, dtype)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(5, 6, 7), (20, 35, 70), (37, 24, 40)])
def test_parity_wide_3d(variant, dtype, shape):
    """General 3D kernels (k3d_wide.cu): Table II 3d13pt (radius-2 star, compile-time point set),
    3d17pt (reading R3e, runtime point list), a reversed 3d7pt list and an asymmetric radius-3 list with random weights (runtime point list):
    every variant bit-exact vs the oracle, ragged 32 x 8 x 8 blocks."""
    _need_gpu()
    o7, _ = si.preset("3d7pt")
    asym = [(0, 0, 0), (3, 0, 0), (-1, 2, 0), (0, -3, 1), (1, 1, -2), (0, 0, 3), (-2, -1, -1)]
    o13, w13 = si.preset("3d13pt")
    o17, w17 = si.preset("3d17pt")
    cases = [(o13, w13), (o17, w17), (o7[::-1], si.random_convex_weights(7, dtype, seed=21)),
             (asym, si.random_convex_weights(len(asym), dtype, seed=22))]
    for offs, w in cases:
        r = max(max(abs(a), abs(b), abs(c)) for a, b, c in offs)
        if min(shape) < 2 * r + 1:
            continue
        u0 = si.field(shape, dtype=dtype, seed=1003)
        for T in (1, 4):
            ref = oracle.run(u0, offs, w, T, nthreads=8)
            _check(_run_gpu_offs(u0, offs, w, T, variant), ref, u0, dtype)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("dtype,shape", [(np.float64, (30, 40, 130)), (np.float32, (33, 50, 136)),
                                         (np.float64, (70, 20, 64)), (np.float32, (9, 17, 256))])
def test_parity_3d13pt_tma_column_kernel(variant, dtype, shape):
    """The TMA column kernel for Table II 3d13pt (k3d_wide.cu unit3t: tensor-box plane loads,
    column registers for the z terms): several tiles and z chunks, ragged x/y tiles, bit-exact vs
    the oracle for every variant (16-byte aligned rows select it)."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset("3d13pt")
    st = Stencil(shape, offs, w, dtype=dtype)
    assert "_tma" in st.query(variant)["kernel"]
    st.close()
    u0 = si.field(shape, dtype=dtype, seed=1313)
    for T in (1, 5):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu(u0, "3d13pt", w, T, variant), ref, u0, dtype)


@pytest.mark.parametrize("name,shape,dtype,variant", [
    ("2d9pt", (300, 520), np.float32, "persistent"),
    ("3d7pt", (24, 40, 64), np.float64, "persistent"),
    ("3d27pt", (20, 36, 128), np.float32, "perks"),
    ("2ds25pt", (200, 300), np.float32, "persistent"),
    ("3d13pt", (20, 24, 64), np.float64, "persistent")])
def test_grid_barrier_counter_wrap(monkeypatch, name, shape, dtype, variant):
    """The device-wide barrier's 32-bit arrival counter wraps modulo 2^32 mid-run (ADVICE r1:
    started just below 2^32 with PERKS_TEST_BAR_BASE) and the run stays bit-exact."""
    _need_gpu()
    monkeypatch.setenv("PERKS_TEST_BAR_BASE", str(2**32 - 700))
    u0 = si.field(shape, dtype=dtype, seed=505)
    offs, w = si.preset(name)
    ref = oracle.run(u0, offs, w, 12, nthreads=4)
    _check(_run_gpu(u0, name, w, 12, variant), ref, u0, dtype)


def test_binding_validates_buffers():
    """The binding rejects buffers whose size/type/device/layout differ from the handle's before
    any raw pointer reaches the library."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200.stencil import run_group
    offs, w = si.preset("2d5pt")
    st = Stencil((16, 16), offs, w, dtype="f64")
    x = torch.ones((16, 16), dtype=torch.float64, device="cuda")
    for bad in (torch.empty((16, 15), dtype=torch.float64, device="cuda"),
                torch.empty((16, 16), dtype=torch.float32, device="cuda"),
                torch.empty((16, 32), dtype=torch.float64, device="cuda")[:, ::2]):
        with pytest.raises(ValueError):
            st.run(x, 1, "hostloop", out=bad)
    with pytest.raises(TypeError):
        st.run(x, 1, "hostloop", out=torch.empty((16, 16), dtype=torch.float64))
    with pytest.raises(ValueError):
        st.run(x.float(), 1, "hostloop")
    with pytest.raises(ValueError):
        st.run_host(np.ones((16, 16), dtype=np.float32), 1)
    with pytest.raises(ValueError):
        st.run_host(np.ones((8, 16), dtype=np.float64), 1)
    with pytest.raises(ValueError):
        st.run_host(np.ones((16, 32), dtype=np.float64)[:, ::2], 1)
    with pytest.raises(TypeError):
        st.run_host(x, 1)
    with pytest.raises(ValueError):
        st.run_host(np.ones((16, 16)), 1, out=np.empty((16, 16), dtype=np.float32))
    with pytest.raises(ValueError):
        run_group([st], [x.float()], 1)
    st.close()


@pytest.mark.parametrize("name", ["3d7pt", "3d27pt", "3d19pt"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("shape", [(3, 3, 3), (9, 17, 33), (34, 40, 132), (37, 24, 128), (64, 48, 100)])
def test_perks3d_resident_bricks(monkeypatch, name, dtype, shape):
    """PERKS-3D resident-brick kernel (opt-in, k3d_brick.cu): the whole domain in shared memory,
    brick surfaces exchanged as tagged words every step; bit-exact for ragged bricks, both step
    parities and back-to-back runs."""
    _need_gpu()
    monkeypatch.setenv("PERKS_P3D_BRICK", "1")
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=dtype)
    q = st.query("perks")
    st.close()
    assert q["kernel"].startswith("perks3d_brick"), q
    u0 = si.field(shape, dtype=dtype, seed=606)
    for T in (1, 2, 7):
        ref = oracle.run(u0, offs, w, T, nthreads=4)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)


@pytest.mark.parametrize("name,dtype", [("2d9pt", np.float32), ("2d5pt", np.float64), ("2ds9pt", np.float32),
                                        ("2d25pt", np.float64)])
@pytest.mark.parametrize("shape", [(700, 900), (517, 1333)])
@pytest.mark.parametrize("tb", ["", "3", "8"])
def test_tiled_perks_2d(monkeypatch, name, dtype, shape, tb):
    """Tiled PERKS ([draft] P:416-441): a domain larger than the (here artificially small: 6 SMs)
    on-chip capacity is cut into device tiles with a redundant halo of r*Tb cells, each advanced Tb
    steps per pass by the resident kernel; bit-exact vs the oracle for step counts that are / are
    not multiples of Tb, both pass parities, ragged tiles."""
    _need_gpu()
    monkeypatch.setenv("PERKS_NUM_SMS", "6")
    if tb:
        monkeypatch.setenv("PERKS_TILED_TB", tb)
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset(name)
    st = Stencil(shape, offs, w, dtype=dtype)
    q = st.query("perks")
    st.close()
    assert q["kernel"].startswith("perks2d_tiled"), q
    u0 = si.field(shape, dtype=dtype, seed=707)
    for T in (1, 7, 16, 17):
        ref = oracle.run(u0, offs, w, T, nthreads=8)
        _check(_run_gpu(u0, name, w, T, "perks"), ref, u0, dtype)
