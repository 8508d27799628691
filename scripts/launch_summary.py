"""Summarises an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    k = r[ki].split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:6d} {v[1] / 1e6:9.3f} ms {v[1] / max(v[0], 1) / 1e3:8.1f} us {100 * v[1] / tot:5.1f}%  {k}")
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
