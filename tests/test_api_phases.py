"""The two PD3 phases and the DRAG phases behind the reference's API
(pardrag.hpp:68-84, drag.hpp:25-28), and MERLIN's length step pinned against
the reference's Eq. 7-8 arithmetic (acceptance criterion 3's range, m=8..512)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def recs_list(recs):
    return [[int(r["index"]), float(r["nn_dist_sq"]).hex()] for r in recs]


def test_par_select_keeps_every_discord_and_refine_is_exact(engine, oracle):
    # tests/pardrag_test.cpp:76-93 ("selection never clears a true range discord")
    x = oracle.gen_randomwalk(600, 5)
    engine.set_series(x)
    m = 8
    nn = oracle.brute_force_nn(x, m)
    s = np.sort(nn)
    for r_sq in (float(s[len(s) * 9 // 10]), float(s[len(s) // 2]), 0.0):
        cand, cnn = engine.par_select(m, r_sq, 32)
        assert np.all(cand[nn >= r_sq] == 1)
        assert np.array_equal(cnn[cand == 1], nn[cand == 1])
        got = engine.par_refine(m, r_sq, 32, cand)
        assert recs_list(got) == recs_list(oracle.range_discords(x, m, r_sq))


def test_par_select_vacuous_threshold(engine, oracle):
    # tests/pardrag_test.cpp:95-106: r = 0 prunes nothing, every nn is finite
    x = oracle.gen_randomwalk(200, 9)
    engine.set_series(x)
    cand, nn = engine.par_select(6, 0.0, 24)
    assert np.all(cand == 1) and np.isfinite(nn[-1])
    assert np.array_equal(nn, oracle.brute_force_nn(x, 6))


def test_par_refine_respects_cleared_candidates(engine, oracle):
    # tests/pardrag_test.cpp:178-189 plus a partial clear
    x = oracle.gen_randomwalk(300, 8)
    engine.set_series(x)
    m = 8
    cand, _ = engine.par_select(m, 4.0 * m + 1.0, 32)
    assert len(engine.par_refine(m, 4.0 * m + 1.0, 32, np.zeros_like(cand))) == 0
    nn = oracle.brute_force_nn(x, m)
    r_sq = float(np.sort(nn)[len(nn) // 2])
    cand, _ = engine.par_select(m, r_sq, 32)
    idx = np.nonzero(cand)[0]
    cand[idx[::2]] = 0
    got = engine.par_refine(m, r_sq, 32, cand)
    want = [r for r in recs_list(oracle.range_discords(x, m, r_sq)) if cand[r[0] - 1]]
    assert recs_list(got) == want


def test_stats_walk_fused_bitexact_to_512(engine, oracle):
    # acceptance criterion 3 (tests/acceptance_test.cpp:157-172): n=10,000 seed 3,
    # m = 8 -> 512, here bit for bit through MERLIN's fused length step
    # (k_next_length with the resident seed rows), not only the plain advance
    x = oracle.gen_randomwalk(10_000, 3)
    engine.set_series(x)
    for m1 in (9, 64, 300, 512):
        mu, sg = engine.stats_walk(8, m1, fused=True)
        omu, osg = oracle.advance_stats(x, 8, m1)
        assert np.array_equal(mu, omu) and np.array_equal(sg, osg), m1
        mu2, sg2 = engine.stats_walk(8, m1, fused=False)
        assert np.array_equal(mu2, omu) and np.array_equal(sg2, osg), m1


def test_stats_walk_offset_series_bitexact(engine, oracle):
    # a DC offset: the same bits as the reference's rolling statistics
    x = oracle.gen_randomwalk(20_000, 4) + 1e5
    engine.set_series(x)
    mu, sg = engine.stats_walk(16, 200, fused=True)
    omu, osg = oracle.advance_stats(x, 16, 200)
    assert np.array_equal(mu, omu) and np.array_equal(sg, osg)


@pytest.mark.parametrize("pk", [0, 1])
def test_resident_seed_rows_follow_the_length_recurrence(engine, oracle, pk):
    # north_star (a): QT_{m+1}(i, q) = QT_m(i, q) + t[i+m] t[q+m] on the device;
    # after 100 steps the rows equal direct FP64 dot products to ~1e-13 relative
    # (the pair-kill band 0 keeps only the positive-side rows, b even, and with
    # its default pattern only the entries its walk reads, u a multiple of 9)
    x = oracle.gen_randomwalk(12_000, 6)
    engine.set_param("pass0_pk", pk)
    try:
        engine.set_series(x)
        m0, m1 = 16, 116
        engine.stats_walk(m0, m1, fused=True)
        info, rows = engine.seed_rows()
    finally:
        engine.set_param("pass0_pk", 1)
    m, L, kA, nb = (int(v) for v in info)
    assert m == m1 and nb > 0
    N = len(x) - m + 1
    worst = 0.0
    for b in range(0, nb, max(1, nb // 7)):
        if pk and (b & 1):
            continue
        j = b >> 1
        i = j * L + L - 1 if (b & 1) else j * L
        if i >= N:
            continue
        for u in ((0, 9, 72, 1143) if pk else (0, 1, 77, 1151)):
            q = i - kA - u if (b & 1) else i + kA + u
            if not (0 <= q < N):
                continue
            direct = float(np.dot(x[i:i + m], x[q:q + m]))
            scale = float(np.dot(np.abs(x[i:i + m]), np.abs(x[q:q + m])))
            worst = max(worst, abs(rows[b, u] - direct) / scale)
    assert worst < 1e-13, worst


def test_cpp_drag_phases_via_pardrag(engine, oracle):
    # drag_select / drag_refine are exposed through the C++ API; their device
    # try is tsd_pardrag: the candidate set equals the range set
    x = oracle.gen_randomwalk(900, 47)
    engine.set_series(x)
    nn = oracle.brute_force_nn(x, 12)
    for q in (0.5, 0.9, 1.0):
        r_sq = float(np.sort(nn)[min(int(len(nn) * q), len(nn) - 1)])
        got = engine.pardrag(12, r_sq, seglen=64)
        assert recs_list(got) == recs_list(oracle.range_discords(x, 12, r_sq))


def periodic_series(n, period=37, seed=5):
    rng = np.random.default_rng(seed)
    x = np.tile(rng.normal(size=period), n // period + 1)[:n].copy()
    x[1000:1005] += 3.0  # one anomaly; every other window has exact repeats (nn = 0)
    return x


def test_overflow_fallback_with_small_caps(engine, oracle):
    # the knife-edge queue and the near-pair buffer overflowing finish the try
    # with the exact pass over the live rows (src/pardrag.cpp:142-149,388-407)
    # instead of failing; thresholds at exact ties make knife edges
    x = oracle.gen_randomwalk(1500, 12)
    engine.set_series(x)
    m = 16
    nn = oracle.brute_force_nn(x, m)
    s = np.sort(nn)
    before = engine.counters()["fallbacks"]
    try:
        for cap in ("queue_cap", "coll_cap"):
            engine.set_param(cap, 1)
            for q in (0.5, 0.9, 0.99):
                r_sq = float(s[int(len(s) * q)])
                got = engine.pardrag(m, r_sq, seglen=64)
                assert recs_list(got) == recs_list(oracle.range_discords(x, m, r_sq)), (cap, q)
            assert np.array_equal(engine.brute_force_nn(m), nn), cap
            engine.set_param(cap, 1 << 30)
    finally:
        engine.set_param("queue_cap", 1 << 30)
        engine.set_param("coll_cap", 1 << 30)
    assert engine.counters()["fallbacks"] > before


def test_periodic_series_merlin_and_bruteforce(engine, oracle):
    # exactly periodic data: thousands of exact ties per row (forced small
    # near-pair buffer so the fallback runs at this size)
    x = periodic_series(4000)
    engine.set_series(x)
    try:
        engine.set_param("coll_cap", 4096)
        assert np.array_equal(engine.brute_force_nn(16), oracle.brute_force_nn(x, 16))
        rep = engine.merlin_full(16, 20, top_k=2, seglen=128)
    finally:
        engine.set_param("coll_cap", 1 << 30)
    exp = oracle.merlin(x, 16, 20, top_k=2, seglen=128)
    for k, m in enumerate(range(16, 21)):
        assert recs_list(rep.per_length[m]) == recs_list(exp["recs"][k][: exp["counts"][k]]), m
    assert np.array_equal(rep.final_r, exp["final_r"]) and np.array_equal(rep.retries, exp["retries"])


@pytest.mark.slow
def test_periodic_series_natural_overflow(engine, oracle):
    # n = 30,000: the near-minimum pairs of brute_force_nn (~N^2 / period = 2.4e7)
    # overflow the 8M buffer at the default capacity
    x = periodic_series(30_000)
    engine.set_series(x)
    before = engine.counters()["fallbacks"]
    assert np.array_equal(engine.brute_force_nn(16), oracle.brute_force_nn(x, 16))
    assert engine.counters()["fallbacks"] > before
