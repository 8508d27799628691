"""Parity of the CUDA path (through the C-ABI) with the reference: golden
fixtures from the unmodified reference, the C oracle on seeded inputs, and
size-independent properties at full size."""
import numpy as np
import pytest

from conftest import hexf, load_golden, series_of

pytestmark = pytest.mark.gpu


def recs_list(recs):
    return [[int(r["index"]), float(r["nn_dist_sq"]).hex(), float(r["nn_dist"]).hex()] for r in recs]


def check_merlin(rep, fx):
    for e in fx["per_length"]:
        m = e["m"]
        assert (m in rep.failed_lengths) == bool(e["failed"]), m
        k = m - fx["min_len"]
        assert float(rep.final_r[k]).hex() == e["final_r"], (m, rep.final_r[k], hexf(e["final_r"]))
        assert int(rep.retries[k]) == e["retries"], m
        if not e["failed"]:
            assert recs_list(rep.per_length[m]) == e["records"], m


# ---- statistics (Eq. 4, Eq. 7-8) -------------------------------------------
def test_stats_bitexact(engine, oracle):
    x = oracle.gen_randomwalk(10_000, 3)
    engine.set_series(x)
    mu, sg = engine.init_stats(8)
    omu, osg = oracle.init_stats(x, 8)
    assert np.array_equal(mu, omu) and np.array_equal(sg, osg)
    for m in range(8, 40):  # acceptance criterion 3, bit-exact instead of 1e-9
        mu, sg = engine.advance_stats(m, mu, sg)
    omu, osg = oracle.advance_stats(x, 8, 40)
    assert np.array_equal(mu, omu) and np.array_equal(sg, osg)


def test_stats_known_answers(engine):
    engine.set_series(np.array([1.0, 2.0, 3.0, 4.0]))
    mu, sg = engine.init_stats(2)
    assert mu.tolist() == [1.5, 2.5, 3.5] and sg.tolist() == [0.5, 0.5, 0.5]


# ---- range discords ----------------------------------------------------------
def test_range_sets_golden(engine):
    g = load_golden("small.json")
    for e in g["range"]:
        engine.set_series(series_of(e["input"]))
        got = engine.pardrag(e["m"], hexf(e["r_sq"]), seglen=max(2 * e["m"], 64))
        assert recs_list(got) == e["records"], (e["input"], e["m"])


@pytest.mark.parametrize("seed", range(6))
def test_range_sets_vs_oracle(engine, oracle, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(300, 3000))
    x = oracle.gen_randomwalk(n, 500 + seed)
    engine.set_series(x)
    for m in (3, 8, 12, 33, 64):
        if 2 * m > n:
            continue
        nn = oracle.brute_force_nn(x, m)
        s = np.sort(nn)
        for q in (0.0, 0.5, 0.9, 0.999, 1.0):
            r_sq = float(s[min(int(len(s) * q), len(s) - 1)]) if q > 0 else 0.0
            exp = oracle.range_discords(x, m, r_sq)
            got = engine.pardrag(m, r_sq, seglen=min(max(2 * m, 64), n))
            assert recs_list(got) == recs_list(exp), (n, m, q)


def test_brute_force_nn_bitexact(engine, oracle):
    x = oracle.gen_randomwalk(1200, 11)
    engine.set_series(x)
    for m in (3, 16, 50):
        assert np.array_equal(engine.brute_force_nn(m), oracle.brute_force_nn(x, m))


def test_series_validation(engine):
    with pytest.raises(ValueError):
        engine.set_series(np.array([1.0, 2.0]))
    with pytest.raises(ValueError):
        engine.set_series(np.array([1.0, np.nan, 2.0, 3.0]))
    engine.set_series(np.arange(100, dtype=float))
    with pytest.raises(ValueError):
        engine.pardrag(2, 1.0, 32)          # m < 3
    with pytest.raises(ValueError):
        engine.pardrag(10, 1.0, 9)          # seglen < m
    with pytest.raises(ValueError):
        engine.merlin_full(10, 60)          # maxL > n/2


# ---- MERLIN --------------------------------------------------------------------
def test_merlin_golden_small(engine):
    for fx in load_golden("small.json")["merlin"]:
        engine.set_series(series_of(fx["input"]))
        rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
        check_merlin(rep, fx)


def test_merlin_golden_c1(engine):
    fx = load_golden("c1.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


def test_merlin_golden_c2(engine):
    fx = load_golden("c2.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


@pytest.mark.parametrize("pair", [0, 1])
def test_merlin_golden_c2_band0_walks(engine, pair):
    # band 0 walked per side (k_scan) and both sides together in packed FP32x2
    # (k_band0_pair, which 512-row blocks enable at this size): same records
    fx = load_golden("c2.json")
    engine.set_series(series_of(fx["input"]))
    engine.set_param("dense_rows", 512)
    engine.set_param("pair_band0", pair)
    try:
        rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
        check_merlin(rep, fx)
    finally:
        engine.set_param("dense_rows", 0)
        engine.set_param("pair_band0", 1)


@pytest.mark.parametrize("knobs", [dict(witness=0, row_cache=0), dict(witness=1, row_cache=0),
                                   dict(witness=0, row_cache=1, rc_min_m=128),
                                   dict(witness=1, row_cache=1, rc_min_m=128, band_few_wit=16)])
def test_merlin_golden_c2_schedule_knobs(engine, knobs):
    # kill witnesses across tries and the row cache only move work between
    # stages: every setting gives the reference's records bit for bit
    fx = load_golden("c2.json")
    engine.set_series(series_of(fx["input"]))
    for k, v in knobs.items():
        engine.set_param(k, v)
    engine.reset_counters()
    try:
        rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
        check_merlin(rep, fx)
        c = engine.counters()
        if knobs["witness"]:
            assert c["wit_kills"] > 0
    finally:
        for k, v in dict(witness=1, row_cache=1, rc_min_m=384, band_few_wit=0).items():
            engine.set_param(k, v)


@pytest.mark.parametrize("knobs", [dict(pass0_pk=0), dict(pass0_pk=1, wit_cache=0),
                                   dict(pass0_pk=1, pk_rows=256, half_pk=1), dict(witness=0, row_cache=0)])
def test_merlin_golden_c3s_schedule_knobs(engine, knobs):
    # n = 5e5 (ECG-like): the pair-kill band 0 (both ends of every pair from one
    # walk), the paired two-sided walk, the witness run-seed cache and other
    # block sizes / strides all give the reference's records bit for bit
    fx = load_golden("c3s.json")
    engine.set_series(series_of(fx["input"]))
    for k, v in knobs.items():
        engine.set_param(k, v)
    try:
        rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
        check_merlin(rep, fx)
    finally:
        for k, v in dict(pass0_pk=1, wit_cache=1, pk_rows=0, half_pk=3, witness=1, row_cache=1).items():
            engine.set_param(k, v)


@pytest.mark.slow
def test_merlin_golden_c4(engine):
    # BASELINE config 4: n=1,000,000 random walk, lengths 512..1024 (513 lengths);
    # the reference needed ~57 min on 6 threads to produce this fixture
    fx = load_golden("c4.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


def test_merlin_golden_c3s(engine):
    # BASELINE config 3 (ECG-like n=500,000), its first 64 lengths (64..127):
    # quasi-periodic data with injected anomalies, the hardest case for pruning
    fx = load_golden("c3s.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


def test_merlin_golden_c3(engine):
    # BASELINE config 3 in full: ECG-like n=500,000, lengths 64..512 (449 lengths;
    # the reference needed 21 min on 6 threads)
    fx = load_golden("c3.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


def test_merlin_golden_c5s(engine):
    # BASELINE config 5 (n=2,000,000 random walk, top-3), its first 32 lengths
    fx = load_golden("c5s.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


@pytest.mark.slow
def test_merlin_golden_c5(engine):
    # BASELINE config 5: n=2,000,000 random walk, lengths 128..640, top-3
    fx = load_golden("c5.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    check_merlin(rep, fx)


def test_merlin_csv_bytes(engine):
    import paper_2304_01660_b200 as P
    g = load_golden("small.json")
    engine.set_series(P.gen_randomwalk(3000, 2024))
    rep = engine.merlin_full(8, 24, top_k=2, seglen=128)
    assert P.discords_csv(rep.per_length) == g["csv_acceptance_c2"]


def test_merlin_vs_oracle_top3(engine, oracle):
    # acceptance criterion 1 shape: single-length top-3 == brute force
    for seed in range(1, 6):
        x = oracle.gen_randomwalk(2000, seed)
        engine.set_series(x)
        for m in (8, 16, 32, 64):
            rep = engine.merlin_full(m, m, top_k=3)
            exp = oracle.merlin(x, m, m, top_k=3)
            assert recs_list(rep.per_length[m]) == recs_list(exp["recs"][0][: exp["counts"][0]])


@pytest.mark.parametrize("seed,paired", [(s, 0) for s in range(1, 9)] + [(s, 1) for s in range(1, 5)])
def test_merlin_random_shapes_vs_oracle(engine, oracle, seed, paired):
    # ragged shapes: n from 600 to 6000 (N below, near and above one tile of
    # 1152 diagonals and 128..512-row blocks), short and long windows, top-1..3;
    # every length's records, final r and retry count equal the C restatement
    rng = np.random.default_rng(seed)
    n = int(rng.integers(600, 6001))
    lo = int(rng.integers(4, 97))
    hi = lo + int(rng.integers(0, 13))
    top_k = int(rng.integers(1, 4))
    x = oracle.gen_randomwalk(n, 100 + seed)
    if seed % 2 == 0:  # a periodic series with noise: many near-equal neighbours
        t = np.arange(n)
        x = np.sin(2 * np.pi * t / (37 + seed)) + 0.05 * x / (np.abs(x).max() + 1.0)
    engine.set_series(x)
    if paired:  # the paired band-0 walk on a series of one or a few (partial) blocks
        engine.set_param("dense_rows", 512)
    try:
        rep = engine.merlin_full(lo, hi, top_k=top_k)
    finally:
        engine.set_param("dense_rows", 0)
    exp = oracle.merlin(x, lo, hi, top_k=top_k)
    for k, m in enumerate(range(lo, hi + 1)):
        assert (m in rep.failed_lengths) == bool(exp["failed"][k]), m
        assert float(rep.final_r[k]) == float(exp["final_r"][k]), m
        assert int(rep.retries[k]) == int(exp["retries"][k]), m
        if not exp["failed"][k]:
            assert recs_list(rep.per_length[m]) == recs_list(exp["recs"][k][: exp["counts"][k]]), m


def test_merlin_constant_series_fails_lengths(engine):
    engine.set_series(np.full(400, 2.5))
    rep = engine.merlin_full(8, 12)
    assert rep.failed_lengths == list(range(8, 13))


# ---- sharded path (segment-sharded tiles + reductions) on one device -----------
@pytest.mark.parametrize("ranks,fused", [(2, 1), (3, 1), (2, 0)])
def test_group_sharded_merlin_equals_single(engine, ranks, fused):
    # ranks contexts on cuda:0: tiles dealt cyclically; kills and route maxima go
    # to every rank's arrays from inside the kernels (fused) or through peer
    # all-reduce kernels; exact-nn keys all-reduced -> identical records
    import paper_2304_01660_b200 as P
    g = P.Group([0] * ranks)
    g.set_param("fused_peers", fused)
    for fx in (load_golden("c1.json"), load_golden("small.json")["merlin"][1]):
        x = series_of(fx["input"])
        g.set_series(x)
        rep = g.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
        check_merlin(rep, fx)
    # every rank swept only its share of the tiles
    cells = [g.counters(r)["cells"] for r in range(ranks)]
    assert all(c > 0 for c in cells)
    g.close()


def test_group_sharded_paired_band0(engine):
    # the paired band-0 walk (k_band0_pair, forced by 512-row blocks) with its
    # row blocks dealt over 2 ranks and fused peer kills: golden C2 records
    import paper_2304_01660_b200 as P
    g = P.Group([0, 0])
    g.set_param("fused_peers", 1)
    g.set_param("dense_rows", 512)
    g.set_param("pair_band0", 1)
    fx = load_golden("c2.json")
    g.set_series(series_of(fx["input"]))
    rep = g.merlin_full(fx["min_len"], fx["min_len"] + 15, top_k=fx["top_k"], seglen=fx["seglen"])
    want = dict(fx)
    want["per_length"] = [e for e in fx["per_length"] if e["m"] <= fx["min_len"] + 15]
    want["max_len"] = fx["min_len"] + 15
    check_merlin(rep, want)
    g.close()


def test_group_sharded_range_sets(engine, oracle):
    import paper_2304_01660_b200 as P
    g = P.Group([0, 0])
    x = oracle.gen_randomwalk(2500, 77)
    g.set_series(x)
    for m in (8, 33):
        s = np.sort(oracle.brute_force_nn(x, m))
        for q in (0.5, 0.99):
            r_sq = float(s[int(len(s) * q)])
            assert recs_list(g.pardrag(m, r_sq, seglen=max(2 * m, 64))) == \
                recs_list(oracle.range_discords(x, m, r_sq))
    g.close()


# ---- independent FP64 matrix profile (STOMP recurrence, no pruning) -------------
def top_k_of(profile, k):
    order = np.lexsort((np.arange(len(profile)), -profile))  # nn desc, index asc (sort_discords)
    return order[:k]


def test_matrix_profile_fp64_vs_reference_bruteforce(engine, oracle):
    for n, m, seed in [(1500, 16, 3), (2400, 64, 9), (900, 100, 4)]:
        x = oracle.gen_randomwalk(n, seed)
        engine.set_series(x)
        mp = engine.matrix_profile_fp64(m)
        bf = oracle.brute_force_nn(x, m)
        assert np.all(np.isfinite(mp) == np.isfinite(bf))
        f = np.isfinite(bf)
        assert np.max(np.abs(mp[f] - bf[f]) / np.maximum(bf[f], 1e-300)) < 1e-9


@pytest.mark.parametrize("name,lengths", [("c4.json", (512, 777, 1024)), ("c3s.json", (64, 100, 127)),
                                          ("c3.json", (300, 512)),
                                          ("c5s.json", (128, 159)), ("c5.json", (384, 640))])
def test_golden_discords_are_matrix_profile_maxima(engine, name, lengths):
    # full-size parity by a second, independent route: the reference's discords of
    # a length are the top-k of the exact nn profile (acceptance criterion 1)
    fx = load_golden(name)
    x = series_of(fx["input"])
    engine.set_series(x)
    per = {e["m"]: e for e in fx["per_length"]}
    for m in lengths:
        e = per[m]
        mp = engine.matrix_profile_fp64(m)
        top = top_k_of(mp, fx["top_k"])
        assert [int(i) + 1 for i in top] == [r[0] for r in e["records"]], m
        for i, r in zip(top, e["records"]):
            assert abs(mp[i] - hexf(r[1])) <= 1e-9 * hexf(r[1]), (m, mp[i], hexf(r[1]))


# ---- constant stretches: the sigma < eps conventions of reference_sq_dist ------
def flat_series(oracle, n, seed, flats):
    x = oracle.gen_randomwalk(n, seed).copy()
    for a, length, level in flats:
        x[a:a + length] = level
    return x


@pytest.mark.parametrize("case", range(4))
def test_constant_stretches_range_sets(engine, oracle, case):
    # exactly constant windows (nrm = 0): d = 0 between two of them, 2m against
    # anything else; they never enter the FP32 band passes and are decided in
    # the full-row stage / survivors with the exact conventions
    rng = np.random.default_rng(40 + case)
    n = int(rng.integers(800, 2500))
    flats = [(int(rng.integers(0, n - 200)), int(rng.integers(20, 120)), float(rng.normal() * 5))
             for _ in range(int(rng.integers(1, 4)))]
    x = flat_series(oracle, n, 900 + case, flats)
    engine.set_series(x)
    for m in (8, 16, 40):
        nn = oracle.brute_force_nn(x, m)
        s = np.sort(nn[np.isfinite(nn)])
        assert np.array_equal(engine.brute_force_nn(m), nn), (case, m)
        for r_sq in (float(s[len(s) // 2]), float(s[-3]), 2.0 * m, 2.0 * m + 1e-9, 1e-12):
            got = engine.pardrag(m, r_sq, seglen=max(2 * m, 64))
            assert recs_list(got) == recs_list(oracle.range_discords(x, m, r_sq)), (case, m, r_sq)


def test_constant_stretches_merlin(engine, oracle):
    x = flat_series(oracle, 3000, 77, [(500, 150, 3.0), (2000, 90, -1.0)])
    engine.set_series(x)
    for top_k in (1, 3):
        rep = engine.merlin_full(8, 24, top_k=top_k, seglen=128)
        exp = oracle.merlin(x, 8, 24, top_k=top_k, seglen=128)
        for k, m in enumerate(range(8, 25)):
            assert (m in rep.failed_lengths) == bool(exp["failed"][k]), m
            if m not in rep.failed_lengths:
                assert recs_list(rep.per_length[m]) == recs_list(exp["recs"][k][: exp["counts"][k]]), m
        assert np.array_equal(rep.final_r, exp["final_r"]) and np.array_equal(rep.retries, exp["retries"])
