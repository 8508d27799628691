"""One MERLIN discovery of a bench config (for ncu launch lists / traces)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_01660_b200 as P
from bench import CONFIGS, make_input

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, seed, lo, hi, top_k, _ = CONFIGS[cfg]
if len(sys.argv) > 2:
    hi = lo + int(sys.argv[2]) - 1
x = make_input(cfg)
e = P.Engine(0)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    e.set_param(k, float(v))
e.set_series(x)
rep = e.merlin_full(lo, hi, top_k=top_k)
c = e.counters()
print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in c.items()})
