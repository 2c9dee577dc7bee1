"""Small CG / SpMV / 3d13pt runs for compute-sanitizer (memcheck, racecheck)."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import seeded_inputs as si, seeded_inputs.sparse as sp
from paper_2204_02064_b200 import CG, Stencil
for dt in ("f64", "f32"):
    ro, ci, va = sp.irregular(3000, mean_degree=8, heavy_rows=2, heavy_degree=300)
    h = CG(ro, ci, va, dtype=dt)
    b = torch.from_numpy(sp.rhs(len(ro) - 1, dtype=np.float64 if dt == "f64" else np.float32)).cuda()
    h.spmv(b)
    for v, p in [("hostloop", "imp"), ("persistent", "imp"), ("perks", "vec"), ("perks", "mat"), ("perks", "mix")]:
        h.solve(b, 6, 0.0, v, p)
    torch.cuda.synchronize()
    h.close()
    shape = (10, 20, 136 if dt == "f32" else 68)
    offs, w = si.preset("3d13pt")
    st = Stencil(shape, offs, w, dtype=np.float64 if dt == "f64" else np.float32)
    x = si.field_torch(shape, np.float64 if dt == "f64" else np.float32, "cuda")
    for v in ("hostloop", "persistent", "perks"):
        st.run(x, 3, v)
    torch.cuda.synchronize()
print("san script ok")
