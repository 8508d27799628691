"""Runs MERLIN on a golden fixture with engine params and lists mismatching lengths.
python scripts/cmp_golden.py c4.json witness=1 band_few_wit=16"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2304_01660_b200 as P
from conftest import load_golden, series_of

fx = load_golden(sys.argv[1])
e = P.Engine(0)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    e.set_param(k, float(v))
e.set_series(series_of(fx["input"]))
rep = e.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
bad = 0
for ent in fx["per_length"]:
    m = ent["m"]
    k = m - fx["min_len"]
    got = [[int(r["index"]), float(r["nn_dist_sq"]).hex()] for r in rep.per_length.get(m, [])]
    want = [[r[0], r[1]] for r in ent["records"]]
    ok = float(rep.final_r[k]).hex() == ent["final_r"] and int(rep.retries[k]) == ent["retries"] and (
        ent["failed"] or got == want)
    if not ok:
        bad += 1
        if bad <= 5:
            print("m", m, "retries", int(rep.retries[k]), ent["retries"], "r", float(rep.final_r[k]),
                  float.fromhex(ent["final_r"]))
            print("   got ", [(i, float.fromhex(h)) for i, h in got][:4])
            print("   want", [(i, float.fromhex(h)) for i, h in want][:4])
print("mismatching lengths:", bad, "of", len(fx["per_length"]), e.counters()["wit_kills"])
