"""Executed-instruction mix of an ncu report's SASS (source page): opcode -> warp instructions,
and stall samples by opcode.  python tools/ncu_opmix.py REP [divisor]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rr = list(csv.reader(src.splitlines()))
hh = rr[1]; rows = rr[2:]
i_s = hh.index('Warp Stall Sampling (All Samples)'); i_src = hh.index('Source'); i_ex = hh.index('Instructions Executed')
ex, sm = collections.Counter(), collections.Counter()
for x in rows:
    t = x[i_src].split()
    if not t: continue
    op = t[1] if t[0].startswith('@') and len(t) > 1 else t[0]
    op = op.split('.')[0]
    ex[op] += int(x[i_ex] or 0); sm[op] += int(x[i_s] or 0)
tot = sum(ex.values())
print(f"total {tot} warp instructions ({tot/div:.2f} per unit), {sum(sm.values())} samples")
for op, n in ex.most_common(30):
    print(f"  {op:10s} {n:>12d} {n/div:8.2f}  samples {sm[op]}")
