"""Record DRAM traffic per launch of the captured kernel into profiles/ncu_traffic.json.

usage: python tools/ncu_traffic.py REPORT.ncu-rep CONFIG T [PLAN_KERNEL]
(REPORT from an ncu capture (--set full, or just the dram__bytes metrics) of one bench-shaped
launch; T = time steps of that launch; PLAN_KERNEL = the plan's kernel name as perks_stencil_query
reports it, which bench.py matches)."""
import csv
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rep, cfg, T = sys.argv[1], sys.argv[2], int(sys.argv[3])
plan_kernel = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
get = lambda k: float(v[h.index(k)].replace(",", "")) * UNIT.get(u[h.index(k)], 1)
name = v[h.index("Kernel Name")]
rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
short = name.split("<")[0].split("::")[-1].replace("void ", "").strip()
d[cfg] = {"kernel": short, "plan_kernel": plan_kernel, "kernel_full": name, "time_steps": T, "dram_read_bytes": rd,
          "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr,
          "dram_bytes_per_step": (rd + wr) / T, "report": os.path.basename(rep)}
json.dump(d, open(path, "w"), indent=1)
print(cfg, d[cfg])
