import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import seeded_inputs.sparse as sp
from paper_2204_02064_b200 import CG
for wl in ["G3", "G5"]:
    kind, size, dtype, iters, _ = sp.CG_WORKLOADS[wl]
    ro, ci, va = sp.matrix(kind, size)
    h = CG(ro, ci, va)
    n = len(ro) - 1
    b = sp.rhs(n)
    bt = torch.from_numpy(b).cuda()
    K = 2000
    for pol in ["mix", "imp", "mat", "vec"]:
        h.solve(bt, K, 0.0, "perks", pol); torch.cuda.synchronize()
        t0 = time.perf_counter(); h.solve(bt, K, 0.0, "perks", pol); torch.cuda.synchronize(); td = time.perf_counter() - t0
        h.solve_host(b, K, 0.0, "perks", pol)
        t0 = time.perf_counter(); h.solve_host(b, K, 0.0, "perks", pol); th = time.perf_counter() - t0
        print(wl, pol, f"device {td*1e3:.2f} ms  host {th*1e3:.2f} ms", flush=True)
