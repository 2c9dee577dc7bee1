"""CG timing sweep (development): us per iteration for each workload x variant/policy, with
CUDA events around one solve of K iterations (tol = 0), best of R."""
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
        if base is None:
            base = t
        gbs = q["unfused_bytes_per_iter"] / (t * 1e-6) / 1e9
        print(f"{wl} {v:10s} {p:4s} {t:9.2f} us/iter  x{base / t:5.2f} vs hostloop  {gbs:8.1f} GB/s unfused "
              f" iters={it} smem={q['smem_per_cta']} cached_nnz={q['cached_nnz_smem']}/{q['nnz']} "
              f"vec_rows={q['cached_rows_smem']} regs={q['regs_per_thread']} tiles={q['tiles']} grid={q['grid']}",
              flush=True)
    h.close()
