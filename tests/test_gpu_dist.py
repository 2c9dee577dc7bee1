"""Multi-GPU slab decomposition (reading R12), emulated on ONE GPU: N slab handles
on cuda:0 exchange their face planes through the same ghost-plane + system-scope counter protocol
(csrc/dist.cuh) that runs over NVLink between GPUs.  The gathered N-slab result must equal the
CPU oracle on the global domain bit-exactly, for several slab counts, step counts of both
parities, and back-to-back runs (which exercises the exchange-parity bookkeeping across runs)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import seeded_inputs as si

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dist(tmp_path, name, shape, dtype, n, variant, Ts):
    out = str(tmp_path / "res.npy")
    env = dict(os.environ)
    if variant == "perks_cache":  # PERKS with the on-chip plane cache tiers (opt-in, k3d_stream.cu)
        variant = "perks"
        env["PERKS_P3D_CACHE"] = "1"
    cmd = [sys.executable, os.path.join(HERE, "dist_worker.py"), out, name, *map(str, shape),
           "f64" if dtype == np.float64 else "f32", str(n), variant, *map(str, Ts)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(out)


@pytest.mark.parametrize("variant", ["hostloop", "persistent", "perks", "perks_cache"])
@pytest.mark.parametrize("n", [2, 3])
@pytest.mark.parametrize("name,dtype", [("3d7pt", np.float64), ("3d27pt", np.float32)])
def test_slabs_match_global_oracle(tmp_path, variant, n, name, dtype):
    _need_gpu()
    shape = (7 * n + 1, 20, 64)  # ragged slabs (nz not a multiple of n)
    offs, w = si.preset(name)
    u0 = si.field(shape, dtype=dtype, seed=505)
    Ts = [3, 4]
    got = _dist(tmp_path, name, shape, dtype, n, variant, Ts)
    ref = oracle.run(u0, offs, w, sum(Ts), nthreads=4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref), f"{int(np.sum(got != ref))} cells differ"


def test_many_slabs_long_run(tmp_path):
    _need_gpu()
    shape, name, dtype = (24, 36, 128), "3d7pt", np.float64
    offs, w = si.preset(name)
    u0 = si.field(shape, dtype=dtype, seed=505)
    ref = oracle.run(u0, offs, w, 16, nthreads=4)
    for variant in ("persistent", "perks", "perks_cache"):
        got = _dist(tmp_path, name, shape, dtype, 4, variant, [1, 10, 5])
        assert np.array_equal(got, ref), variant


def test_two_process_ipc_slabs(tmp_path):
    """Two PROCESSES on one GPU, one z-slab each: the neighbour's ghost planes are mapped with
    cudaIpcOpenMemHandle (the cross-process exchange path, api.cu), host-loop variant (each step's
    kernel waits only for the neighbour's face counter, so time-sliced processes make progress).
    The gathered result equals the global oracle bit-exactly."""
    _need_gpu()
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    shape, name, dtype = (17, 24, 64), "3d7pt", np.float64
    prefix = str(tmp_path / "slab")
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        cmd = [sys.executable, os.path.join(HERE, "dist_ipc_worker.py"), prefix, name,
               *map(str, shape), "f64", "hostloop", "3", "2"]
        procs.append(subprocess.Popen(cmd, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True))
    logs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        logs.append(out)
        assert p.returncode == 0, "\n".join(logs)
    got = np.concatenate([np.load(f"{prefix}{r}.npy") for r in range(2)], axis=0)
    offs, w = si.preset(name)
    ref = oracle.run(si.field(shape, dtype=dtype, seed=505), offs, w, 5, nthreads=4)
    assert np.array_equal(got, ref), f"{int(np.sum(got != ref))} cells differ"


@pytest.mark.parametrize("n", [2, 3])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_slabs_two_steps_per_pass(tmp_path, n, dtype):
    """The 7-point star's slab plan is the two-steps-per-pass kernel (k3d_tb.cu): two-deep ghost planes
    exchanged once per pass, the neighbours' planes -1 / nz computed redundantly.  Bit-exact vs the
    global oracle for odd / even T, and with one-step-per-pass runs interleaved on the same handles
    (exchange bookkeeping in plane units, separate ghost planes)."""
    _need_gpu()
    from paper_2204_02064_b200 import Stencil
    offs, w = si.preset("3d7pt")
    st = Stencil((9, 40, 64), offs, w, dtype=dtype, rank=0, nranks=n)
    q = st.query("perks")
    st.close()
    assert q["kernel"].startswith("perks3d_tb2"), q
    shape = (9 * n + 2, 40, 64)
    u0 = si.field(shape, dtype=dtype, seed=505)  # (dist_worker.py seeds the global field with 505)
    Ts = [5, 4, 3, 6]
    got = _dist(tmp_path, "3d7pt", shape, dtype, n, "perks,persistent,perks,hostloop", Ts)
    ref = oracle.run(u0, offs, w, sum(Ts), nthreads=4)
    assert not np.isnan(got).any()
    assert np.array_equal(got, ref), f"{int(np.sum(got != ref))} cells differ"


def test_slabs_two_deep_ghosts_minimum_planes(tmp_path):
    """Slabs of 2 and 3 planes: a face plane goes to both neighbours in the same pass."""
    _need_gpu()
    offs, w = si.preset("3d7pt")
    shape = (7, 24, 64)  # slab_bounds(7, 3): 3 / 2 / 2 planes
    u0 = si.field(shape, dtype=np.float64, seed=505)
    Ts = [4, 5]
    got = _dist(tmp_path, "3d7pt", shape, np.float64, 3, "perks", Ts)
    ref = oracle.run(u0, offs, w, sum(Ts), nthreads=4)
    assert np.array_equal(got, ref), f"{int(np.sum(got != ref))} cells differ"
