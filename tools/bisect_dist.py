import os, subprocess, sys
import numpy as np
sys.path.insert(0, '.')
import oracle, seeded_inputs as si
offs, w = si.preset("3d7pt")
shape = (20, 40, 64)
u0 = si.field(shape, dtype=np.float64, seed=505)
for seq, Ts in [("perks", [5, 4]), ("perks,persistent", [5, 4]), ("persistent,perks", [5, 4]), ("perks,hostloop", [5, 4]),
                ("hostloop,perks", [4, 5]), ("perks,persistent,perks", [4, 4, 4]), ("persistent,persistent", [5, 4])]:
    out = "/tmp/res.npy"
    r = subprocess.run([sys.executable, "tests/dist_worker.py", out, "3d7pt", *map(str, shape), "f64", "2", seq, *map(str, Ts)],
                       capture_output=True, text=True, timeout=300)
    if r.returncode:
        print(seq, Ts, "FAIL rc", r.stderr[-300:]); continue
    got = np.load(out)
    ref = oracle.run(u0, offs, w, sum(Ts), nthreads=8)
    bad = got != ref
    zs = sorted(set(np.nonzero(bad)[0].tolist()))
    print(seq, Ts, "bad cells", int(bad.sum()), "planes", zs[:20])
