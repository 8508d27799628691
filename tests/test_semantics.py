"""Reference semantics the long goldens never reach (tests/golden/semantics.json,
made by the unmodified reference through tests/golden/make_golden.py):

* the retry budget: exhaustion accepts a non-empty list and fails an empty one
  (/root/reference/proj/src/merlin.cpp:104-107);
* reuse_stats = false (tests/merlin_test.cpp:80-99): init_stats per length;
* a failed warm-up length leaves fewer than 5 history entries at the first
  steady length, so ThresholdHistory::window_mean throws std::logic_error
  through merlin (src/merlin.cpp:19,77-82);
* DC offsets: |mean| >> sigma stresses the rolling statistics and the FP32
  filter (the reference stays self-consistent there);
* acceptance criterion 10's case study, top-6 (tests/golden/c10.json).

The CPU tests pin the C oracle to the same fixtures; the gpu tests run the
CUDA path through the C-ABI."""
import numpy as np
import pytest

from conftest import hexf, load_golden, series_of


def recs_list(recs):
    return [[int(r["index"]), float(r["nn_dist_sq"]).hex(), float(r["nn_dist"]).hex()] for r in recs]


def cases():
    return load_golden("semantics.json")


def _check(failed, final_r, retries, per_length, fx):
    for k, e in enumerate(fx["per_length"]):
        m = e["m"]
        assert bool(failed(k)) == bool(e["failed"]), m
        assert float(final_r[k]).hex() == e["final_r"], (m, final_r[k], hexf(e["final_r"]))
        assert int(retries[k]) == e["retries"], m
        if not e["failed"]:
            assert recs_list(per_length(k)) == e["records"], m


def test_semantics_fixture_shape():
    names = [c["name"] for c in cases()]
    for want in ("max_retries_0", "max_retries_1", "max_retries_2", "logic_error_77_17",
                 "reuse_stats_0", "offset_100000_3000", "offset_1e+05_c1"):
        assert want in names
    assert any(c.get("error") for c in cases())


@pytest.mark.parametrize("idx", range(14))
def test_oracle_semantics(oracle, idx):
    from oracle.refbind import CheckerError
    cs = cases()
    if idx >= len(cs):
        pytest.skip("no such case")
    fx = cs[idx]
    x = series_of(fx["input"])
    kw = dict(top_k=fx["top_k"], seglen=fx["seglen"], max_retries=fx["max_retries"],
              reuse_stats=fx["reuse_stats"])
    if fx.get("error"):
        with pytest.raises(CheckerError) as ei:
            oracle.merlin(x, fx["min_len"], fx["max_len"], **kw)
        assert ei.value.code == fx["error"]["code"] and fx["error"]["message"] in str(ei.value)
        return
    if fx["n"] >= 10_000:  # the O(N^2 m) oracle: first lengths only (CPU budget)
        fx = dict(fx, max_len=fx["min_len"] + 2, per_length=fx["per_length"][:3])
    out = oracle.merlin(x, fx["min_len"], fx["max_len"], **kw)
    _check(lambda k: out["failed"][k], out["final_r"], out["retries"],
           lambda k: out["recs"][k][: out["counts"][k]], fx)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(14))
def test_gpu_semantics(engine, idx):
    import paper_2304_01660_b200 as P
    cs = cases()
    if idx >= len(cs):
        pytest.skip("no such case")
    fx = cs[idx]
    engine.set_series(series_of(fx["input"]))
    kw = dict(top_k=fx["top_k"], seglen=fx["seglen"], max_retries=fx["max_retries"],
              reuse_stats=fx["reuse_stats"])
    if fx.get("error"):
        with pytest.raises(P.LogicError) as ei:
            engine.merlin_full(fx["min_len"], fx["max_len"], **kw)
        assert fx["error"]["message"] in str(ei.value)
        return
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], **kw)
    ms = list(range(fx["min_len"], fx["max_len"] + 1))
    _check(lambda k: ms[k] in rep.failed_lengths, rep.final_r, rep.retries,
           lambda k: rep.per_length[ms[k]], fx)


@pytest.mark.gpu
def test_gpu_offset_series_vs_oracle(engine, oracle):
    # larger DC offsets than the fixtures, against the brute-force contract on
    # single lengths (every record of the range set, two thresholds)
    for off in (3e4, 1e5, 3e5):
        x = oracle.gen_randomwalk(2500, 99) + off
        engine.set_series(x)
        for m in (8, 24, 64):
            nn = oracle.brute_force_nn(x, m)
            s = np.sort(nn)
            for q in (0.5, 0.97):
                r_sq = float(s[int(len(s) * q)])
                got = engine.pardrag(m, r_sq, seglen=max(2 * m, 64))
                assert recs_list(got) == recs_list(oracle.range_discords(x, m, r_sq)), (off, m, q)


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_criterion10_top6(engine):
    # acceptance criterion 10's case study (n=35,040, lengths 48-672, top-6)
    fx = load_golden("c10.json")
    engine.set_series(series_of(fx["input"]))
    rep = engine.merlin_full(fx["min_len"], fx["max_len"], top_k=fx["top_k"], seglen=fx["seglen"])
    ms = list(range(fx["min_len"], fx["max_len"] + 1))
    assert not rep.failed_lengths
    _check(lambda k: ms[k] in rep.failed_lengths, rep.final_r, rep.retries,
           lambda k: rep.per_length[ms[k]], fx)
