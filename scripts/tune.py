"""Parameter sweep of one MERLIN discovery: python scripts/tune.py c2 dense_rows=256,512 ..."""
import sys
import os
import itertools

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_01660_b200 as P
from bench import CONFIGS, make_input

cfg = sys.argv[1]
n, seed, lo, hi, top_k, _ = CONFIGS[cfg]
grid = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    grid[k] = [float(x) for x in v.split(",")]
x = make_input(cfg)
e = P.Engine(0)
e.set_series(x)
e.merlin_full(lo, hi, top_k=top_k)  # warm
base = None
for combo in itertools.product(*grid.values()) if grid else [()]:
    for k, v in zip(grid.keys(), combo):
        e.set_param(k, v)
    best = None
    for _ in range(3):
        e.reset_counters()
        rep = e.merlin_full(lo, hi, top_k=top_k)
        c = e.counters()
        if best is None or c["total_ms"] < best["total_ms"]:
            best = c
    key = [(r["index"].tolist(), r["nn_dist_sq"].tolist()) for r in rep.per_length.values()]
    same = base is None or key == base
    base = base or key
    c = best
    print(dict(zip(grid.keys(), combo)), f"total {c['total_ms']:.2f} ms scan {c['scan_ms']:.2f} dense {c['dense_ms']:.2f} "
          f"sparse {c['sparse_ms']:.2f} collect {c['collect_ms']:.2f} syncs {c['host_syncs']} "
          f"launches {c['kernel_launches']} seeds {c['seed_dots']} wit {c['wit_kills']}/{c['wit_tests']} same={same}", flush=True)
