"""Generates the committed golden fixtures in tests/golden/ by running the
UNMODIFIED reference library (oracle/_ref/libtsdref.so, built from
/root/reference/proj/src by `make -C oracle ref`).  Run in the build container:

    python tests/golden/make_golden.py small          # seconds
    python tests/golden/make_golden.py c1 c2          # C1 ~2 s, C2 ~1 min (8 threads)
    python tests/golden/make_golden.py c4 --workers 8 # ~40 min: full-size parity
    python tests/golden/make_golden.py semantics      # retry budget, reuse_stats, logic_error, offsets
    python tests/golden/make_golden.py c10            # acceptance criterion 10 shape, top-6

Every fixture stores the inputs (generator + seed, or the literal series), the
call, and the reference's outputs, so tests can check both the C restatement
(oracle/oracle.c) and the CUDA library against them without /root/reference.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.refbind import CheckerError, Ref  # noqa: E402

CONFIGS = {
    # c3: BASELINE config 3 (ECG-like n=500,000, lengths 64-512); "c3s" is its first
    # 64 lengths, the parity fixture that fits the build container's CPU budget
    "c3": (500_000, 1, 64, 512, 1, 512),
    "c3s": (500_000, 1, 64, 127, 1, 512),
    # name: (n, seed, minL, maxL, top_k, seglen)   (BASELINE.json configs)
    "c1": (10_000, 1, 64, 128, 1, 512),
    "c2": (100_000, 1, 128, 256, 1, 512),
    "c4": (1_000_000, 1, 512, 1024, 1, 512),
    "c5": (2_000_000, 1, 128, 640, 3, 512),
    # "c5s": the first 32 lengths of C5 (top-3), the parity fixture that fits the
    # build container's CPU budget
    "c5s": (2_000_000, 1, 128, 159, 3, 512),
    # acceptance criterion 10's case study (tests/acceptance_test.cpp:410-446): top-6
    "c10": (35_040, 1048, 48, 672, 6, 512),
}


def recs_to_list(recs):
    return [[int(r["index"]), float(r["nn_dist_sq"]).hex(), float(r["nn_dist"]).hex()] for r in recs]


def merlin_fixture(R, x, gen, minL, maxL, top_k, seglen, workers, max_retries=100,
                   reuse_stats=True):
    t = time.time()
    try:
        out = R.merlin(x, minL, maxL, top_k=top_k, seglen=seglen, workers=workers,
                       max_retries=max_retries, reuse_stats=reuse_stats)
    except CheckerError as e:  # the reference threw (e.g. logic_error from src/merlin.cpp:19)
        return dict(kind="merlin", input=gen, n=len(x), min_len=minL, max_len=maxL, top_k=top_k,
                    seglen=seglen, max_retries=max_retries, reuse_stats=reuse_stats,
                    error=dict(code=e.code, message=str(e).split("] ", 1)[1]))
    dt = time.time() - t
    per = []
    for k in range(maxL - minL + 1):
        per.append(dict(m=minL + k, failed=int(out["failed"][k]), final_r=float(out["final_r"][k]).hex(),
                        retries=int(out["retries"][k]),
                        records=recs_to_list(out["recs"][k][: out["counts"][k]])))
    return dict(kind="merlin", input=gen, n=len(x), min_len=minL, max_len=maxL, top_k=top_k,
                seglen=seglen, max_retries=max_retries, reuse_stats=reuse_stats, ref_seconds=dt,
                ref_workers=workers, per_length=per)


def small(R):
    fx = {}
    # generator pins (src/io.cpp:110-119)
    fx["randomwalk"] = []
    for n, seed in [(10_000, 1), (1000, 7), (100_000, 3), (5, 0)]:
        x = R.gen_randomwalk(n, seed)
        fx["randomwalk"].append(dict(n=n, seed=seed, head=[v.hex() for v in x[:8].tolist()],
                                     last=x[-1].hex(), sum=float(np.sum(x)).hex()))
    # stats literals (tests/stats_test.cpp:14-28) + recurrence through m=8..64
    x = R.gen_randomwalk(3000, 3)
    mu, sg = R.advance_stats(x, 8, 64)
    fx["stats"] = dict(input=dict(gen="randomwalk", n=3000, seed=3), m0=8, m1=64,
                       mu_head=[v.hex() for v in mu[:16].tolist()],
                       sigma_head=[v.hex() for v in sg[:16].tolist()],
                       mu_sum=float(np.sum(mu)).hex(), sigma_sum=float(np.sum(sg)).hex())
    # brute-force nn profiles and range sets (pardrag == {nn >= r^2})
    fx["range"] = []
    rng = np.random.default_rng(2304)
    for inst in range(12):
        n = int(rng.integers(300, 1600))
        m = int([8, 12, 16, 32][inst % 4])
        seed = 1000 + inst
        x = R.gen_randomwalk(n, seed)
        nn = R.brute_force_nn(x, m)
        s = np.sort(nn)
        for q in (0.5, 0.95):
            r_sq = float(s[int(len(s) * q)])
            recs = R.pardrag(x, m, r_sq, seglen=max(2 * m, 64), workers=4)
            fx["range"].append(dict(input=dict(gen="randomwalk", n=n, seed=seed), m=m,
                                    r_sq=r_sq.hex(), records=recs_to_list(recs)))
    # merlin cases from the reference tests
    fx["merlin"] = [
        # tests/merlin_test.cpp:47-63 (n=2000 seed 123, m 8..32, top-1, seglen 64)
        merlin_fixture(R, R.gen_randomwalk(2000, 123), dict(gen="randomwalk", n=2000, seed=123),
                       8, 32, 1, 64, 4),
        # tests/acceptance_test.cpp:134-151 (n=3000 seed 2024, m 8..24, top-2, seglen 128)
        merlin_fixture(R, R.gen_randomwalk(3000, 2024), dict(gen="randomwalk", n=3000, seed=2024),
                       8, 24, 2, 128, 4),
        # acceptance criterion 1 style (n=2000, single length, top-3)
        merlin_fixture(R, R.gen_randomwalk(2000, 7), dict(gen="randomwalk", n=2000, seed=7),
                       32, 32, 3, 512, 4),
    ]
    fx["csv_acceptance_c2"] = R.merlin_csv(R.gen_randomwalk(3000, 2024), 8, 24, top_k=2,
                                           seglen=128, workers=4)
    # heatmap / ranking of that discord CSV (the reference CLI's `heatmap` outputs)
    import hashlib
    hm = {}
    for name, csv, n in [("acceptance_c2", fx["csv_acceptance_c2"], 3000)]:
        hm[name] = dict(n=n, heatmap_csv_sha256=hashlib.sha256(R.heatmap(csv, n, 10, 0)).hexdigest(),
                        pgm_sha256=hashlib.sha256(R.heatmap(csv, n, 10, 1)).hexdigest(),
                        ranking_csv=R.heatmap(csv, n, 10, 2).decode(),
                        ranking_k3=R.heatmap(csv, n, 3, 2).decode())
    fx["heatmap"] = hm
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(fx, f, indent=0)
    print("wrote small.json")


def semantics(R):
    """Reference-semantics cases the long goldens never reach:
    the retry budget (src/merlin.cpp:104-107), reuse_stats=false (tests/merlin_test.cpp:80-99),
    a warm-up failure that makes the steady phase throw logic_error (src/merlin.cpp:19,77-82),
    and series with a DC offset (the rolling statistics and the FP32 filter see |mean| >> sigma)."""
    fx = []

    def walk(n, seed, offset=0.0):
        x = R.gen_randomwalk(n, seed) + offset
        g = dict(gen="randomwalk", n=n, seed=seed)
        if offset:
            g["offset"] = offset
        return x, g

    # retry budget: exhaustion accepts a non-empty list, an empty one fails the length
    for mr in (0, 1, 2):
        x, g = walk(2000, 5)
        fx.append(dict(name=f"max_retries_{mr}", **merlin_fixture(R, x, g, 8, 20, 3, 64, 4, max_retries=mr)))
        x, g = walk(77, 17)
        fx.append(dict(name=f"max_retries_{mr}_short", **merlin_fixture(R, x, g, 4, 8, 1, 16, 1, max_retries=mr)))
    # warm-up failure: a failed warm-up length leaves < 5 history entries at the first
    # steady length -> ThresholdHistory::window_mean throws std::logic_error
    for n, seed, minL in ((77, 17, 4), (69, 9, 6)):
        x, g = walk(n, seed)
        fx.append(dict(name=f"logic_error_{n}_{seed}", **merlin_fixture(R, x, g, minL, minL + 9, 1, 16, 1, max_retries=2)))
    # reuse_stats = false (tests/merlin_test.cpp:80-99 shape) and true for comparison
    for reuse in (False, True):
        x, g = walk(1200, 55)
        fx.append(dict(name=f"reuse_stats_{int(reuse)}", **merlin_fixture(R, x, g, 8, 24, 2, 48, 4, reuse_stats=reuse)))
    # DC offsets: the reference stays self-consistent (== brute force) up to ~3e5 here
    for off in (1e4, 1e5):
        x, g = walk(3000, 2024, off)
        fx.append(dict(name=f"offset_{off:g}_3000", **merlin_fixture(R, x, g, 8, 24, 2, 128, 4)))
    x, g = walk(10000, 1, 1e5)
    fx.append(dict(name="offset_1e+05_c1", **merlin_fixture(R, x, g, 64, 128, 1, 512, 8)))
    with open(os.path.join(HERE, "semantics.json"), "w") as f:
        json.dump(fx, f, indent=0)
    print("wrote semantics.json")


def big(R, name, workers):
    n, seed, minL, maxL, top_k, seglen = CONFIGS[name]
    if name.startswith("c3"):
        from paper_2304_01660_b200.datasets import gen_ecg_like
        x = gen_ecg_like(n, seed)
        spec = dict(gen="ecg", n=n, seed=seed, sha256=hashlib.sha256(x.tobytes()).hexdigest())
    else:
        x = R.gen_randomwalk(n, seed)
        spec = dict(gen="randomwalk", n=n, seed=seed)
    fx = merlin_fixture(R, x, spec, minL, maxL, top_k, seglen, workers)
    fx["config"] = name
    with open(os.path.join(HERE, f"{name}.json"), "w") as f:
        json.dump(fx, f, indent=0)
    print(f"wrote {name}.json in {fx['ref_seconds']:.1f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="+")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    R = Ref()
    for w in a.what:
        if w == "small":
            small(R)
        elif w == "semantics":
            semantics(R)
        else:
            big(R, w, a.workers)
