"""CG timing sweep (development): us per iteration for each workload x variant/policy, with
CUDA events around one solve of K iterations (tol = 0), best of R."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import seeded_inputs.sparse as sp  # noqa: E402
from paper_2204_02064_b200 import CG  # noqa: E402

wls = sys.argv[1].split(",") if len(sys.argv) > 1 else ["G2", "G3", "G4", "G5"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
combos = [("hostloop", "imp"), ("persistent", "imp"), ("perks", "vec"), ("perks", "mat"), ("perks", "mix")]
for wl in wls:
    kind, size, dtype, _, desc = sp.CG_WORKLOADS[wl]
    ro, ci, va = sp.matrix(kind, size)
    n = len(ro) - 1
    h = CG(ro, ci, va, dtype="f64" if dtype == np.float64 else "f32")
    b = torch.from_numpy(sp.rhs(n, dtype=dtype)).cuda()
    base = None
    y = torch.empty_like(b)
    h.spmv(b, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        h.spmv(b, out=y)
    e1.record()
    torch.cuda.synchronize()
    t_sp = e0.elapsed_time(e1) * 1e3 / 20
    mb = (h.nnz * (8 if dtype == np.float64 else 4) + h.nnz * 4 + (n + 1) * 4 + 2 * n * (8 if dtype == np.float64 else 4))
    print(f"{wl} spmv kernel {t_sp:9.2f} us  {mb / t_sp / 1e3:8.1f} GB/s (A + x + y once)", flush=True)
    for v, p in combos:
        q = h.query(v, p)
        x, hist, info = h.solve(b, 3, 0.0, v, p)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, hist, info = h.solve(b, K, 0.0, v, p, out=x, history=hist if hist.numel() > K else None)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / K)
        it = int(info[0].item())
        t = min(ts)
        phases = ""
        if os.environ.get("PERKS_CG_TIMING") and v != "hostloop":
            ws = h.workspace()
            ws[256:256 + 8 * 528].zero_()
            h.solve(b, K, 0.0, v, p, out=x, history=hist)
            torch.cuda.synchronize()
            d = ws[256:256 + 8 * 528].cpu().numpy().view(np.uint64)
            nit = max(int(d[8]), 1)
            g = q["grid"]
            per = d[16:16 + g] / nit / 1e3
            phases = (" phases(us/iter): " + " ".join(f"{d[i] / nit / 1e3:.2f}" for i in range(4)) +
                      f" spmv/CTA min {per.min():.2f} med {np.median(per):.2f} max {per.max():.2f}"
                      f" argmax {int(per.argmax())}")
        if base is None:
            base = t
        gbs = q["unfused_bytes_per_iter"] / (t * 1e-6) / 1e9
        print(f"{wl} {v:10s} {p:4s} {t:9.2f} us/iter  x{base / t:5.2f} vs hostloop  {gbs:8.1f} GB/s unfused "
              f" iters={it} smem={q['smem_per_cta']} cached tm/sm={q['cached_nnz_tmem']}/{q['cached_nnz_smem']} of {q['nnz']} ({q['tmem_tiles_per_cta']}+{q['smem_tiles_per_cta']} tiles) "
              f"vec_rows={q['cached_rows_smem']} regs={q['regs_per_thread']} tiles={q['tiles']} grid={q['grid']}{phases}",
              flush=True)
    h.close()
