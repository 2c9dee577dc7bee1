"""Timing of the general 3D kernels (k3d_wide.cu) on Table II 3d13pt: host loop / persistent / PERKS."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, seeded_inputs as si
from paper_2204_02064_b200 import Stencil
for name, dt, shp in [("3d13pt", np.float64, (256,256,256)), ("3d13pt", np.float32, (512,512,512))]:
  offs,w=si.preset(name)
  for v in ["hostloop","persistent","perks"]:
    st=Stencil(shp,offs,w,dtype=dt); x=si.field_torch(shp,dt,"cuda"); out=torch.empty_like(x); ws=st.workspace(v)
    st.run(x,5,v,out=out,workspace=ws); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record(); st.run(x,100,v,out=out,workspace=ws); e1.record(); torch.cuda.synchronize()
    us=e0.elapsed_time(e1)*1000/100; S=x.element_size(); cells=np.prod(shp)
    print(name, np.dtype(dt).name, shp[0], v, st.query(v)["kernel"], st.query(v)["grid"], "%.2f us/step  %.0f GB/s"%(us, 2*S*cells/us/1e3))
