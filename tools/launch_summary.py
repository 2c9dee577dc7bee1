"""Summarise ncu launch lists (--metrics gpu__time_duration.sum --csv): per kernel name, total time,
share and launch count.  python tools/launch_summary.py TITLE=FILE.csv ..."""
import collections
import csv
import sys

print("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 launch lists of the bench command")
print("# (cold-cache, serialised: compare SHARES, not absolutes)")
for arg in sys.argv[1:]:
    title, path = arg.split("=", 1)
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if r]
    hdr = rows[0]
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] in ("ns", "nsecond") else v * 1e3 if r[iu] in ("ms", "msecond") else v
        tot[r[ik]] += v
        cnt[r[ik]] += 1
    s = sum(tot.values())
    print(f"\n== {title}")
    for k, v in tot.most_common(8):
        print(f"  {v:10.1f} us {100 * v / s:6.1f}%  x{cnt[k]:<3d} {k[:100]}")
