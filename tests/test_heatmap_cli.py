"""Heatmap / ranking on the device and the command-line front end, against the
reference's own outputs (tests/golden/small.json: `heatmap`, produced by the
unmodified reference via oracle/ref_shim.cpp: tsdref_heatmap)."""
import hashlib
import math
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden

CLI = os.path.join(ROOT, "paper_2304_01660_b200", "tsdiscord")


def heatmap_csv(scores) -> bytes:
    import paper_2304_01660_b200 as P
    return "".join(",".join(P.format_double(v) for v in row) + "\n" for row in scores).encode()


def heatmap_pgm(scores) -> bytes:
    rows, cols = scores.shape
    px = bytes(int(math.floor(min(max(v / 2.0, 0.0), 1.0) * 255.0 + 0.5)) for v in scores.ravel())
    return f"P5\n{cols} {rows}\n255\n".encode() + px


def test_read_discords_csv_roundtrip():
    import paper_2304_01660_b200 as P
    g = load_golden("small.json")
    d = P.read_discords_csv(g["csv_acceptance_c2"])
    assert P.discords_csv(d) == g["csv_acceptance_c2"]
    with pytest.raises(RuntimeError):
        P.read_discords_csv("index,length\n1,2\n")


def test_cli_usage_and_gen_rw(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    import paper_2304_01660_b200 as P
    r = subprocess.run([CLI, "discover", "--input", "x"], capture_output=True, text=True)
    assert r.returncode == 106 and "required" in r.stderr
    out = tmp_path / "rw.txt"
    subprocess.run([CLI, "gen-rw", "--n", "1000", "--seed", "7", "--output", str(out)], check=True)
    got = np.array([float(v) for v in out.read_text().split()])
    assert np.array_equal(got, P.gen_randomwalk(1000, 7))
    pin = [e for e in load_golden("small.json")["randomwalk"] if e["n"] == 1000 and e["seed"] == 7][0]
    assert [v.hex() for v in got[:8]] == pin["head"]


@pytest.mark.gpu
def test_heatmap_and_ranking_match_reference(engine):
    import paper_2304_01660_b200 as P
    g = load_golden("small.json")
    fx = g["heatmap"]["acceptance_c2"]
    d = P.read_discords_csv(g["csv_acceptance_c2"])
    sc = engine.heatmap(d, fx["n"], scores=True)
    assert hashlib.sha256(heatmap_csv(sc)).hexdigest() == fx["heatmap_csv_sha256"]
    assert hashlib.sha256(heatmap_pgm(sc)).hexdigest() == fx["pgm_sha256"]
    assert P.ranking_csv(engine.heatmap_rank(10)) == fx["ranking_csv"]
    assert P.ranking_csv(engine.heatmap_rank(3)) == fx["ranking_k3"]
    # host-edited matrix: the device column max follows the upload
    sc[0, 0] = 1.75
    engine.heatmap_set(sc, min(d), max(d), fx["n"])
    top = engine.heatmap_rank(1)
    assert int(top[0]["index"]) == 1 and float(top[0]["score"]) == 1.75 and int(top[0]["length"]) == min(d)
    with pytest.raises(ValueError):
        engine.heatmap_rank(0)
    with pytest.raises(ValueError):
        engine.heatmap(d, 20)  # maxL >= n


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    g = load_golden("small.json")
    series = tmp_path / "s.txt"
    subprocess.run([CLI, "gen-rw", "--n", "3000", "--seed", "2024", "--output", str(series)], check=True)
    out = tmp_path / "d.csv"
    r = subprocess.run([CLI, "discover", "--input", str(series), "--minl", "8", "--maxl", "24", "--topk", "2",
                        "--seglen", "128", "--output", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert out.read_text() == g["csv_acceptance_c2"]
    assert "length 8: 2 discord(s)" in r.stdout
    r = subprocess.run([CLI, "oracle-check", "--input", str(series), "--minl", "8", "--maxl", "12", "--topk", "2",
                        "--discords", str(out)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.count("PASS") == 5, r.stdout
    pre = tmp_path / "hm"
    r = subprocess.run([CLI, "heatmap", "--input", str(out), "--n", "3000", "--output", str(pre)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    fx = g["heatmap"]["acceptance_c2"]
    assert hashlib.sha256((tmp_path / "hm_heatmap.csv").read_bytes()).hexdigest() == fx["heatmap_csv_sha256"]
    assert hashlib.sha256((tmp_path / "hm_heatmap.pgm").read_bytes()).hexdigest() == fx["pgm_sha256"]
    assert (tmp_path / "hm_ranking.csv").read_text() == fx["ranking_csv"]
