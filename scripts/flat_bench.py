"""Flat-stretch cost (degenerate windows): one MERLIN discovery of
C2 (n=1e5 random walk, lengths 128-256) as is, and with a constant stretch of
600 samples at level 0 (every window one-pass constant: the O(1) conventions)
and at a non-zero level (about half the windows have tiny equal z: exact pairs).
Device time per discovery, best of 3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_01660_b200 as P

x0 = P.gen_randomwalk(100_000, 1)
e = P.Engine(0)
for name, level in (("plain", None), ("flat@0", 0.0), ("flat@3.7", 3.7)):
    x = x0.copy()
    if level is not None:
        x[50_000:50_600] = level
    e.set_series(x)
    best = None
    for _ in range(3):
        e.reset_counters()
        rep = e.merlin_full(128, 256, top_k=1)
        ms = e.counters()["total_ms"]
        best = ms if best is None else min(best, ms)
    c = e.counters()
    top = [(m, int(rep.per_length[m][0]["index"]), float(rep.per_length[m][0]["nn_dist_sq"]))
           for m in (128, 192, 256) if m in rep.per_length]
    print(f"{name:10s} {best:9.2f} ms  tries {c['pardrag_calls']}  top {top}", flush=True)
