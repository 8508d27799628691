"""Runs one C2 discovery with TSD_DEBUG=1 (per-pass trace on stderr) and prints counters."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_01660_b200 as P
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, lo, hi = {"c2": (100_000, 128, 256), "c1": (10_000, 64, 128), "c4": (1_000_000, 512, 1024)}[cfg]
if len(sys.argv) > 2:
    hi = lo + int(sys.argv[2]) - 1
e = P.Engine(0)
e.set_series(P.gen_randomwalk(n, 1))
e.merlin_full(lo, min(hi, lo + 2))
e.reset_counters()
t = time.time()
rep = e.merlin_full(lo, hi)
print("wall", time.time() - t, file=sys.stderr)
print(e.counters(), file=sys.stderr)
e.close()
