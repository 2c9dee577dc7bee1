"""C2's PERKS tile (256x256 fp32 9pt, cfg 0) on 1, 4, 9, 36, 144 tiles: how much of the per-step time is the
inter-tile exchange?  (PERKS_P2D_CFG=0 forces the tile; T=1000)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PERKS_P2D_CFG"] = "0"
import numpy as np, torch
import seeded_inputs as si
from paper_2204_02064_b200 import Stencil
offs, w = si.preset("2d9pt")
for n in [256, 512, 768, 1536, 3072]:
    st = Stencil((n, n), offs, w, dtype=np.float32)
    x = si.field_torch((n, n), np.float32, "cuda")
    out = torch.empty_like(x)
    ws = st.workspace("perks")
    st.run(x, 100, "perks", out=out, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st.run(x, 1000, "perks", out=out, workspace=ws); e1.record(); torch.cuda.synchronize()
    q = st.query("perks")
    print(f"{n}x{n} tiles={q['grid']} {q['kernel']} {e0.elapsed_time(e1):.3f} us/step")
