"""bench.py — the driver's benchmark contract for the PERKS stencil library on B200.

One bench "step" = one pass of the whole hot path: perks_stencil_run over the full time loop
(T time steps) of the configured workload.  Default: C4 = BASELINE.json configs[3], 3D 27-point
box stencil fp32 512^3, T=500 — BASELINE.json's metric names no config, so the headline is the
largest configuration that fits one GPU (C5 is the multi-GPU slab workload; C1-C3 and C5 are
selectable with --config and are parity-test cases, not the headline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--config C1..C5|G1..G5] [--variant perks|persistent|hostloop|auto]
                    [--policy auto|imp|vec|mat|mix]

--config G1..G5 benches the PERKS conjugate-gradient workloads with the
paper's CG metric, sustained GB/s; see run_cg.

Prints ONE JSON line on rank 0.  `value` = whole-job GCell-updates/s (cells x T x K x N / max
over ranks of the device-timed region).  `--impl reference` times the CPU oracle (the only other
place bench.py executes oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import seeded_inputs as si  # noqa: E402

METRIC = "stencil GCell-updates/s & effective HBM GB/s vs peak; speedup over host-loop"
UNIT = "GCells/s"
FP32_FMA_PER_CLK_SM = 128   # B200 SM: 4 SMSPs x 32 FP32 lanes
FP64_FMA_PER_CLK_SM = 64    # B200 FP64: half the FP32 rate
CONFIG_DESC = {
    "C1": "2D 5-point Jacobi fp64 128x128, T=100",
    "C2": "2D 9-point box fp32 3072x3072, T=1000",
    "C3": "3D 7-point heat fp64 256^3, T=1000",
    "C4": "3D 27-point box fp32 512^3, T=500",
    "C5": "3D 7-point fp64 1024^3 per GPU, T=100",
}


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        med = statistics.median(sm) if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cfg(name):
    c = dict(si.CONFIGS[name])
    c["np_dtype"] = np.float64 if c["dtype"] == "f64" else np.float32
    c["cells"] = int(np.prod(c["shape"]))
    c["S"] = 8 if c["dtype"] == "f64" else 4
    return c


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    """CPU oracle, as it stands, on a bounded sample of the workload (rank 0 only)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle

    c = _cfg(args.config)
    offs, w = si.preset(c["stencil"])
    cores = os.cpu_count() or 1
    u0 = si.field(c["shape"], dtype=c["np_dtype"])
    # bounded sample: T_s time steps of the full domain, sized to ~2-4 s per bench step
    flops_cell = 2 * len(offs)
    t0 = time.perf_counter()
    oracle.run(u0, offs, w, 1, nthreads=cores)
    t1 = time.perf_counter() - t0
    T_s = int(max(1, min(c["steps"], 3.0 / max(t1, 1e-6))))
    for _ in range(args.warmup):
        oracle.run(u0, offs, w, 1, nthreads=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.run(u0, offs, w, T_s, nthreads=cores)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = c["cells"] * T_s * args.steps / tot / 1e9
    sample = (f"{CONFIG_DESC[args.config]}: full domain, {T_s} of {c['steps']} time steps per "
              f"bench step, {cores} OpenMP threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}", "sample_steps": T_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": sample, "flops_per_cell": flops_cell},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm

def cpu_baseline(c, budget_s=12.0, budget_1t_s=6.0):
    """Oracle timed on the host cores on a bounded sample (rank 0, N=1 only): all cores
    (OpenMP over rows) and one thread (the plain, slow oracle), SURVEY §8(d)."""
    import oracle

    offs, w = si.preset(c["stencil"])
    cores = os.cpu_count() or 1
    u0 = si.field(c["shape"], dtype=c["np_dtype"])
    t0 = time.perf_counter()
    oracle.run(u0, offs, w, 1, nthreads=cores)
    t1 = max(time.perf_counter() - t0, 1e-6)
    T_s = int(max(1, min(c["steps"], budget_s / t1)))
    t0 = time.perf_counter()
    oracle.run(u0, offs, w, T_s, nthreads=cores)
    dt = time.perf_counter() - t0
    # one thread: a slab of the domain's slowest axis (rows/planes 0..k), one time step, sized to
    # about budget_1t_s from the all-core rate (the oracle's per-cell cost is size independent)
    per_cell_1t = dt * cores / (c["cells"] * T_s)  # estimate, refined by the measurement itself
    n0 = c["shape"][0]
    k = int(max(3, min(n0, budget_1t_s / max(per_cell_1t * c["cells"] / n0, 1e-12))))
    sub = np.ascontiguousarray(u0[:k])
    t0 = time.perf_counter()
    oracle.run(sub, offs, w, 1, nthreads=1)
    dt1 = time.perf_counter() - t0
    cells1 = int(np.prod(sub.shape))
    return {"value": c["cells"] * T_s / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"full domain, {T_s} of {c['steps']} time steps, {cores} OpenMP threads, "
                      f"{dt:.1f} s",
            "single_thread": {"value": cells1 / dt1 / 1e9, "unit": UNIT, "cores": 1,
                              "sample": f"{k} of {n0} slowest-axis slices x 1 time step, 1 thread, "
                                        f"{dt1:.1f} s"}}


def _traffic_from_profiles(kernel_prefix, config):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        e = d.get(config, {})
        if e.get("plan_kernel") == kernel_prefix or (not e.get("plan_kernel") and
                                                      e.get("kernel", "").startswith(kernel_prefix.split("_")[0])):
            return e.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


def run_nccl_slab(args):
    """SURVEY §8(e)(a) baseline: C5 z-slabs, face planes exchanged every step by NCCL send/recv
    (torch.distributed batch_isend_irecv), one host-loop step per time step through the C ABI
    (paper_2204_02064_b200/nccl_slab.py).  Same metric/config as the in-kernel exchange path."""
    import torch
    import torch.distributed as tdist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if ws > 1:
        tdist.init_process_group("nccl", device_id=dev)
    from paper_2204_02064_b200 import Stencil
    from paper_2204_02064_b200.nccl_slab import NcclSlabHostLoop

    c = _cfg(args.config)
    offs, w = si.preset(c["stencil"])
    T = args.T or c["steps"]
    nz, ny, nx = c["shape"]
    nzg = nz * ws
    radius = max(max(abs(v) for v in o) for o in offs)
    holder = {}

    def empty(shape):
        return torch.empty(shape, dtype=torch.float64 if c["dtype"] == "f64" else torch.float32, device=dev)

    def step(src, dst):
        st = holder.get("st")
        if st is None:
            st = holder["st"] = Stencil(tuple(src.shape), offs, w, dtype=c["np_dtype"], device=local)
            holder["ws"] = st.workspace("hostloop")
        st.run(src, 1, "hostloop", out=dst, workspace=holder["ws"])

    sl = NcclSlabHostLoop((nzg, ny, nx), radius, rank, ws, step, empty)
    sl.load(si.field_torch((sl.nz, ny, nx), c["np_dtype"], dev, index_offset=sl.z0 * ny * nx))
    sl.run(1)
    for _ in range(args.warmup):
        sl.run(T)
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream(dev)
    per = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sl.run(T)
        e1.record(stream)
        torch.cuda.synchronize()
        per.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    tot_ms = sum(per)
    if ws > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms = float(t.item())
    cells = nz * ny * nx
    value = cells * T * args.steps * ws / (tot_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}, global z = {nz} x {ws}",
                   "parallelism": f"slab{ws}", "variant": "nccl-hostloop",
                   "exchange": "per step: ncclSend/ncclRecv of the face planes (torch.distributed "
                               "batch_isend_irecv), then one host-loop kernel on the halo-extended slab",
                   "time_steps_per_bench_step": T},
        "us_per_time_step": 1e3 * tot_ms / args.steps / T,
        "gpu_launches": T * args.steps, "clocks": clocks, "e2e": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def run_mine(args):
    import torch

    ws, rank, local = _dist()
    dist = ws > 1
    if dist:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2204_02064_b200 import Stencil

    c = _cfg(args.config)
    offs, w = si.preset(c["stencil"])
    T = args.T or c["steps"]
    # C5 is the slab-decomposed workload: rank r owns global planes [r*nz, (r+1)*nz) of a
    # 1024 x 1024 x (1024*N) domain and exchanges face planes with its neighbours every step
    # (in-kernel, csrc/dist.cuh).  Every other config runs independent replicas at N > 1.
    slab = args.config == "C5" and ws > 1
    if slab:
        st = Stencil(c["shape"], offs, w, dtype=c["np_dtype"], device=local, rank=rank, nranks=ws)
        st.connect_torch_distributed()
    else:
        st = Stencil(c["shape"], offs, w, dtype=c["np_dtype"], device=local)
    x = si.field_torch(c["shape"], c["np_dtype"], dev,
                       index_offset=(rank * c["cells"]) if slab else 0)
    out = torch.empty_like(x)
    variant = args.variant
    q = st.query(variant)
    wsp = st.workspace(variant)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MiB L2

    def one(v, wsv):
        st.run(x, T, v, out=out, workspace=wsv)

    for _ in range(args.warmup):
        one(variant, wsp)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ev = []
    for _ in range(args.steps):
        flush.fill_(1)  # L2 flush between timed steps (outside the timed interval)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one(variant, wsp)
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    clocks = sampler.stop()
    per = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(per)
    best_ms, med_ms = min(per), statistics.median(per)
    if dist:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms = float(t.item())
    cells, S = c["cells"], c["S"]
    value = cells * T * args.steps * ws / (tot_ms * 1e-3) / 1e9
    ms_per = tot_ms / args.steps

    # --- host-loop reference variant of the same library, same workload (speedup over host loop)
    hl = None
    if variant != "hostloop" and not args.no_hostloop:
        wsh = st.workspace("hostloop")
        one("hostloop", wsh)
        torch.cuda.synchronize()
        hts = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one("hostloop", wsh)
            e1.record(stream)
            torch.cuda.synchronize()
            hts.append(e0.elapsed_time(e1))
        hl = statistics.mean(hts)

    # --- end to end through the public API with host buffers (H2D + run + D2H per step)
    e2e = None
    if not args.no_e2e:
        hin = torch.empty(c["shape"], dtype=x.dtype, pin_memory=True)
        hin.copy_(x.cpu())
        hout = torch.empty_like(hin).pin_memory()
        st.run_host(hin, T, variant, out=hout)  # warm (allocates the handle's device buffers)
        n_e2e = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            st.run_host(hin, T, variant, out=hout)
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            dt = float(t.item())
        nbytes = cells * S
        e2e = {"value": cells * T * n_e2e * ws / dt / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "timing": "host wall clock around perks_stencil_run_host (pinned host buffers)"}

    # --- roofline of the dominant kernel (the one launch per step for PERKS / persistent)
    peaks = _peaks()
    npts = len(offs)
    tb2 = q["kernel"].startswith("perks3d_tb2")  # PERKS-3D, two time steps per pass
    launches_per_step = st.launch_count(variant, T)
    kern_ms = ms_per / max(1, launches_per_step)
    if q["variant"] == "perks" and c["stencil"].startswith("2d"):
        # fully resident domain: on-chip FMA bound
        fma_rate = FP32_FMA_PER_CLK_SM if c["dtype"] == "f32" else FP64_FMA_PER_CLK_SM
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = 2.0 * fma_rate * sms * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        flops = 2.0 * npts * cells * T / max(1, launches_per_step)
        achieved = flops / (kern_ms * 1e-3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "peak_source": "derived: SMs x FMA/clk x 2 x sm_max_mhz"}
    else:
        # HBM bound: algorithmic bytes = model A_gm per launch (2·S·cells·T·(1-f) + 2·S·D_cache);
        # two steps per pass (k3d_tb.cu): S·cells per step (perks_stencil_info.dram_bytes_per_step)
        f = ((q["cached_cells_reg"] + q["cached_cells_smem"] + q["cached_cells_tmem"]) / cells
             if q["variant"] == "perks" else 0.0)
        if tb2:
            alg = q["dram_bytes_per_step"] * T / max(1, launches_per_step)
        else:
            alg = (2.0 * S * cells * (1 - f) * T + 2.0 * S * cells * f) / max(1, launches_per_step)
        achieved = alg / (kern_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof["traffic"] = _traffic_from_profiles(q["kernel"], args.config)
    roof["kernel"] = q["kernel"]

    eff_gbs = 2.0 * S * cells * T * args.steps * ws / (tot_ms * 1e-3) / 1e9
    from paper_2204_02064_b200 import model

    cached = (q["cached_cells_reg"] + q["cached_cells_smem"] + q["cached_cells_tmem"]
              if q["variant"] == "perks" else 0)
    # ℙ (Eq. maxpeak) with T_sm (Eq. time_sm): D^sm_cache = the cells the plan
    # keeps in shared memory, A_sm(KERNEL) = the kernel's own shared-memory accesses per cell and
    # step (the paper's small-domain example counts 4): 3D plane streaming = one TMA write +
    # the (R+2)(V+2)/(R·V) neighbourhood reads of each cell; the 2D tile kernels keep x/y
    # neighbours in registers/shuffles (edge columns only, ~0).  B_sm = SMs x 128 B/clk x the SM
    # clock sampled under load (P:495 convention, 108 x 128 B x 1.41 GHz on A100).
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_sm = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)) * 1e6
    B_sm = model.b_sm(sms, 128, f_sm)
    if tb2:
        # per two steps: the TMA box write ((TY+4)(TX+2·PAD)/(TX·TY)), stage-1 neighbourhood reads
        # (rows (R+2)/R, x-neighbours 2/V), the IS write, stage-2 reads (own rows from registers:
        # x-neighbours 2/V of R rows + 2 full rows), halved per step
        V, R = (4, 4) if S == 4 else (2, 4)
        TX, TY, PAD = 32 * V, 8 * R, 16 // S
        k_box = (TY + 4) * (TX + 2 * PAD) / (TX * TY)
        k_s1 = (R + 2) / R * (V + 2) / V
        k_s2 = (2.0 / V) + 2.0 / R * (V + 2) / V
        k_sm = 0.5 * (k_box + k_s1 + 1.0 + k_s2)
    elif c["stencil"].startswith("3d"):
        V, R = (4, 2) if S == 4 else (2, 2)
        k_sm = 1.0 + (R + 2) * (V + 2) / (R * V)
    else:
        k_sm = 0.0
    D_sm = min(q["cached_cells_smem"], cells) if q["variant"] == "perks" else 0
    proj = model.project(cells, min(cached, cells), T, S, peaks["hbm_gbs"] * 1e9,
                         A_halo=q["halo_bytes_per_step"] / S * T, D_sm_cache=D_sm, B_sm=B_sm,
                         A_sm_kernel=k_sm * cells * T,
                         A_gm_elems=(cells * T if tb2 else None))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
        "config": {
            "parallelism": (f"slab{ws}" if slab else f"replicas{ws}") if ws > 1 else "single",
            "workload": f"{args.config}: {CONFIG_DESC[args.config]}"
                        + ((f", global z = 1024 x {ws}, slab-decomposed, face planes exchanged "
                            "in-kernel every step" if slab else " per GPU (independent replicas)")
                           if ws > 1 else ""),
            "variant": q["variant"], "kernel": q["kernel"], "grid": q["grid"], "block": q["block"],
            "time_steps_per_bench_step": T, "cells": cells,
            "l2": "flushed between timed steps (256 MiB device write outside the events)",
            "inputs": "seeded splitmix64 field in [1,2), dyadic preset weights",
        },
        "effective_gbs": eff_gbs,
        "hbm_frac_effective": eff_gbs / ws / peaks["hbm_gbs"],
        "us_per_time_step": 1e3 * ms_per / T,
        "hostloop_ms_per_step": hl,
        "speedup_vs_hostloop": (hl / ms_per) if hl else None,
        "ms_per_step_best": best_ms, "ms_per_step_median": med_ms,
        "model": {"P_gcells": proj.peak_cells_per_s / 1e9,
                  "M_over_P": (value / ws) / (proj.peak_cells_per_s / 1e9),
                  "T_gm_s": proj.t_gm, "T_halo_s": proj.t_halo, "T_sm_s": proj.t_sm,
                  "D_sm_cache": int(D_sm), "A_sm_kernel_per_cell_step": k_sm,
                  "B_sm_gbs": B_sm / 1e9,
                  "ref": "P:519 A_gm, P:565-571 T_sm, P:578-584 T_halo, P:587-603 T_PERKS, P"},
        "roofline": roof,
        "gpu_launches": int(launches_per_step * args.steps),
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(c)
    if rank == 0:
        print(json.dumps(line), flush=True)
    st.close()
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- CG (NEXT-3)
# --config G1..G5: the PERKS conjugate-gradient workloads (seeded_inputs/sparse.py CG_WORKLOADS,
# the Table V size classes).  One bench step = one solve of K iterations (tol = 0) from x0 = 0.
# Metric: the paper's CG figure of merit, sustained memory bandwidth: unfused-equivalent
# bytes per iteration (matrix in CSR once + the 15 vector accesses per row of Algorithm P:244-258,
# perks_cg_info.unfused_bytes_per_iter) x iterations / time.
CG_METRIC = "CG sustained GB/s (unfused-equivalent bytes per iteration, P:465); speedup over host-loop"


def _cg_setup(name):
    import seeded_inputs.sparse as sp

    kind, size, dtype, iters, desc = sp.CG_WORKLOADS[name]
    ro, ci, va = sp.matrix(kind, size)
    return sp, kind, size, dtype, iters, desc, ro, ci, va


def _cg_oracle_rate(ro, ci, va, b, iters, unfused, budget_s, nthreads):
    import oracle

    oracle.cg(ro, ci, va, b, kmax=1, nthreads=nthreads)  # warm (thread pool, library load)
    t0 = time.perf_counter()
    oracle.cg(ro, ci, va, b, kmax=1, nthreads=nthreads)
    t1 = max(time.perf_counter() - t0, 1e-6)
    k = int(max(1, min(iters, budget_s / t1)))
    t0 = time.perf_counter()
    _, _, kk = oracle.cg(ro, ci, va, b, kmax=k, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return unfused * kk / dt / 1e9, kk, dt


def run_cg_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    sp, kind, size, dtype, iters, desc, ro, ci, va = _cg_setup(args.config)
    n, nnz = len(ro) - 1, len(ci)
    S = 8 if dtype == np.float64 else 4
    unfused = nnz * (S + 4) + (n + 1) * 4 + n * S * 15
    b = sp.rhs(n, dtype=dtype)
    cores = os.cpu_count() or 1
    times, ks = [], []
    for i in range(args.warmup + args.steps):
        v, kk, dt = _cg_oracle_rate(ro, ci, va, b, iters, unfused, 2.0, cores)
        if i >= args.warmup:
            times.append(dt)
            ks.append(kk)
    value = unfused * sum(ks) / sum(times) / 1e9
    line = {
        "impl": "reference", "metric": CG_METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if dtype == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", "sample_iterations": ks[0]},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{ks[0]} of {iters} CG iterations per bench step, {cores} OpenMP threads "
                                   "(SpMV rows in parallel, inner products sequential)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_cg(args):
    import torch

    ws, rank, local = _dist()
    dist = ws > 1
    if dist:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    from paper_2204_02064_b200 import CG

    sp, kind, size, dtype, iters, desc, ro, ci, va = _cg_setup(args.config)
    K = args.T or iters
    n, nnz = len(ro) - 1, len(ci)
    h = CG(ro, ci, va, dtype="f64" if dtype == np.float64 else "f32", device=local)
    b = torch.from_numpy(sp.rhs(n, dtype=dtype)).to(dev)
    x = torch.empty_like(b)
    hist = torch.empty(K + 1, dtype=torch.float64, device=dev)
    info = torch.zeros(2, dtype=torch.int64, device=dev)
    variant = args.variant if args.variant != "auto" else "perks"
    policy = args.policy
    q = h.query(variant, policy)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one(v, p):
        h.solve(b, K, 0.0, v, p, out=x, history=hist, info=info)

    for _ in range(args.warmup):
        one(variant, policy)
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ev = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        one(variant, policy)
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    clocks = sampler.stop()
    done = int(info[0].item())
    per = [a.elapsed_time(c) for a, c in ev]
    tot_ms = sum(per)
    if dist:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per = tot_ms / args.steps
    unfused = q["unfused_bytes_per_iter"]
    value = unfused * done * args.steps * ws / (tot_ms * 1e-3) / 1e9
    hl = None
    if variant != "hostloop" and not args.no_hostloop:
        one("hostloop", "imp")
        torch.cuda.synchronize()
        hts = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one("hostloop", "imp")
            e1.record(stream)
            torch.cuda.synchronize()
            hts.append(e0.elapsed_time(e1))
        hl = statistics.mean(hts)
    e2e = None
    if not args.no_e2e:
        bh = sp.rhs(n, dtype=dtype)
        h.solve_host(bh, K, 0.0, variant, policy)
        n_e2e = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            _, _, kk, _ = h.solve_host(bh, K, 0.0, variant, policy)
        dt = time.perf_counter() - t0
        S = 8 if dtype == np.float64 else 4
        e2e = {"value": unfused * kk * n_e2e * ws / dt / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": n * S, "d2h_bytes_per_step": n * S + (K + 1) * 8 + 16,
               "timing": "host wall clock around perks_cg_solve_host (b in, x + history + info out)"}
    peaks = _peaks()
    launches = 1 if variant != "hostloop" else 2 * K + 2
    kern_ms = ms_per / launches
    alg = q["dram_bytes_per_iter"] * done / launches
    achieved = alg / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "peak_source": "MEASURED_PEAKS.json hbm_gbs",
            "traffic": None, "kernel": q["kernel_name"],
            "algorithmic_bytes": "modelled DRAM bytes per iteration (uncached matrix tiles + vectors "
                                 "leaving the SM), perks_cg_info.dram_bytes_per_iter"}
    line = {
        "metric": CG_METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if dtype == np.float64 else "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", "iterations_per_bench_step": done,
                   "variant": q["variant"], "policy": q["policy"], "kernel": q["kernel_name"],
                   "grid": q["grid"], "block": q["block"], "n_rows": n, "nnz": nnz,
                   "cached_items_tmem": q["cached_nnz_tmem"], "cached_items_smem": q["cached_nnz_smem"],
                   "parallelism": f"replicas{ws}" if ws > 1 else "single",
                   "l2": "flushed between timed steps (256 MiB device write outside the events)"},
        "us_per_iteration": 1e3 * ms_per / max(done, 1),
        "hostloop_ms_per_step": hl, "speedup_vs_hostloop": (hl / ms_per) if hl else None,
        "ms_per_step_best": min(per), "ms_per_step_median": statistics.median(per),
        "roofline": roof, "gpu_launches": launches * args.steps, "clocks": clocks, "e2e": e2e,
    }
    if rank == 0 and ws == 1 and not args.no_cpu:
        bh = sp.rhs(n, dtype=dtype)
        cores = os.cpu_count() or 1
        v, kk, dt = _cg_oracle_rate(ro, ci, va, bh, K, unfused, 8.0, cores)
        v1, kk1, dt1 = _cg_oracle_rate(ro, ci, va, bh, K, unfused, 4.0, 1)
        line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                                "sample": f"{kk} of {K} iterations, {cores} OpenMP threads, {dt:.1f} s",
                                "single_thread": {"value": v1, "unit": "GB/s", "cores": 1,
                                                  "sample": f"{kk1} of {K} iterations, 1 thread, {dt1:.1f} s"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    h.close()
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(si.CONFIGS) + ["G1", "G2", "G3", "G4", "G5"],
                    help="C5 = the slab-decomposed multi-GPU workload (N>1 under torchrun); "
                         "G1..G5 = the PERKS CG workloads (NEXT-3)")
    ap.add_argument("--policy", default="auto", choices=["auto", "imp", "vec", "mat", "mix"],
                    help="CG cache policy (G configs)")
    ap.add_argument("--variant", default="perks",
                    choices=["perks", "persistent", "hostloop", "auto", "nccl"],
                    help="nccl = the NCCL host-loop slab baseline (C5, SURVEY §8(e)(a))")
    ap.add_argument("--T", type=int, default=0, help="override time steps (dev only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hostloop", action="store_true")
    args = ap.parse_args()
    if args.config.startswith("G"):
        return run_cg_reference(args) if args.impl == "reference" else run_cg(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.variant == "nccl":
        return run_nccl_slab(args)
    return run_mine(args)


if __name__ == "__main__":
    sys.exit(main())
