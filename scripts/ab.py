"""A/B timing of library builds: python scripts/ab.py c4 ab/libA.so ab/libB.so [key=val ...]
Each build runs in its own process, 3 discoveries, alternating twice; prints the best total_ms."""
import os
import subprocess
import sys

cfg, libs = sys.argv[1], [a for a in sys.argv[2:] if a.endswith(".so")]
kv = [a for a in sys.argv[2:] if "=" in a]
code = r'''
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2304_01660_b200 as P
from bench import CONFIGS, make_input
n, seed, lo, hi, top_k, _ = CONFIGS[sys.argv[1]]
e = P.Engine(0)
for a in sys.argv[2:]:
    k, v = a.split("="); e.set_param(k, float(v))
e.set_series(make_input(sys.argv[1]))
e.merlin_full(lo, hi, top_k=top_k)
best = 1e30
for _ in range(3):
    e.reset_counters(); e.merlin_full(lo, hi, top_k=top_k); best = min(best, e.counters()["total_ms"])
print(best)
'''
res = {l: [] for l in libs}
for rep in range(2):
    for l in libs:
        out = subprocess.run([sys.executable, "-c", code, cfg, *kv], env={**os.environ, "TSD_LIB": os.path.abspath(l)},
                             capture_output=True, text=True)
        res[l].append(float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else float("nan"))
        if out.returncode:
            print(out.stderr[-500:])
for l, v in res.items():
    print(f"{l}: {' '.join(f'{x:.2f}' for x in v)} ms")
