"""Per-CUDA-source-line instruction counts and stall samples from an ncu report
(cuda,sass source view).  Usage: ncu_lines.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, path = [], None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        if r[0] == "Line No":
            hdr = r
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if r[2] != "-":  # SASS rows carry an address; the CUDA-line rows carry aggregates
        continue
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    rows.append((ie, ss, f"{path}:{ln}", r[1].strip()[:70]))
tot_i = sum(x[0] for x in rows)
tot_s = sum(x[1] for x in rows)
print(f"total instructions {tot_i}  samples {tot_s}")
key = (lambda x: x[1]) if "--samples" in sys.argv else (lambda x: x[0])
for ie, ss, where, src in sorted(rows, key=key, reverse=True)[:n]:
    print(f"{ie:>11} {100*ie/max(tot_i,1):5.1f}% {ss:>6} {where:24s} {src}")
