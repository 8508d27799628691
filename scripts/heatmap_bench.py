"""Heatmap / ranking on the device at C4 size: build the
513 x 999,488 FP64 score matrix (4.1 GB) from the C4 discords and time the
HBM-bound column-max pass of rank_discords against the measured HBM peak.
Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2304_01660_b200 as P  # noqa: E402

fx = json.load(open(os.path.join(ROOT, "tests", "golden", "c4.json")))
per = {e["m"]: np.array([(r[0], float.fromhex(r[1]), float.fromhex(r[2])) for r in e["records"]],
                        dtype=P.RECORD_DTYPE) for e in fx["per_length"] if not e["failed"]}
n, lo, hi = fx["n"], fx["min_len"], fx["max_len"]
e = P.Engine(0)
t0 = time.perf_counter()
e.heatmap(per, n, lo, hi, scores=False)
build_s = time.perf_counter() - t0
times = []
for _ in range(5):
    rk = e.heatmap_rank(10)
    times.append(e.counters()["heatmap_ms"])
ms = min(times)
rows, cols = hi - lo + 1, n - lo
bytes_read = rows * cols * 8
peak = None
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
gbs = bytes_read / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": "k_hm_colmax", "matrix": [rows, cols], "bytes": bytes_read, "ms": ms,
                  "achieved_gbs": gbs, "peak_gbs": peak, "frac": (gbs / peak) if peak else None,
                  "build_s_incl_scatter": build_s, "top": [[int(r["index"]), int(r["length"]), float(r["score"])]
                                                          for r in rk[:3]]}))
