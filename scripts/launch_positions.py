"""Per-stage breakdown of an ncu launch list: the n-th launch of each kernel within a DRAG try."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = [(r[ki].split("(")[0].replace("tsd::", "").replace("void ", ""), float(r[vi].replace(",", ""))) for r in rows[1:]]
start = sys.argv[2] if len(sys.argv) > 2 else "k_try_init"
tries, cur = [], None
for k, v in seq:
    if k == start:
        cur = []
        tries.append(cur)
    if cur is not None:
        cur.append((k, v))
pos = collections.defaultdict(list)
for t in tries:
    c = collections.Counter()
    for k, v in t:
        c[k] += 1
        pos[(k, c[k])].append(v)
for (k, i), vs in sorted(pos.items(), key=lambda x: -sum(x[1]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    vs.sort()
    print(f"{k:22s} #{i}  n={len(vs):4d} sum={sum(vs) / 1e6:7.3f}ms med={vs[len(vs) // 2] / 1e3:7.1f}us "
          f"max={vs[-1] / 1e3:8.1f}us")
