"""load_series (src/io.cpp:48-104) of the library against the unmodified
reference on the same files: same values, same exception kinds and messages.
Host-only (no GPU): both drivers are built here from tests/cpp/."""
import os
import subprocess

import pytest

from conftest import ROOT

PKG = os.path.join(ROOT, "paper_2304_01660_b200")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtsdref.so")
CASES = {
    "plain.txt": "1.5\n-2\n3e-3\n\n4\n",
    "crlf.txt": "1\r\n2\r\n3\r\n",
    "hdr.csv": "time,value,other\n0, 1.25 ,x\n1,2.5,y\n2,3.75,z\n",
    "nohdr.csv": "5,6\n7,8\n9,10\n",
    "badnum.csv": "a,b\n1,2\n3,x\n5,6\n",
    "missing.csv": "1,2\n3\n5,6\n",
    "short.txt": "1\n2\n",
    "blank_lines.txt": "\n\n 1 \n\t2\n\n3\n",
    "nan.txt": "1\nnan\n3\n",
    "trailing_comma.csv": "1,\n2,\n3,\n",
}
ARGS = [("plain.txt", "-"), ("crlf.txt", "-"), ("hdr.csv", "value"), ("hdr.csv", "1"), ("hdr.csv", "nope"),
        ("nohdr.csv", "1"), ("nohdr.csv", "value"), ("badnum.csv", "b"), ("missing.csv", "1"),
        ("short.txt", "-"), ("blank_lines.txt", "-"), ("nan.txt", "-"), ("trailing_comma.csv", "1"),
        ("does_not_exist.txt", "-")]


def build(tmp, lib_dir, lib_name, include, out):
    subprocess.run(["g++", "-std=gnu++20", "-O1", "-I", include, "-include", "cstdint",
                    os.path.join(ROOT, "tests", "cpp", "load_series_driver.cpp"), "-L", lib_dir, "-l" + lib_name,
                    "-Wl,-rpath," + lib_dir, "-o", out], check=True, capture_output=True)


def run(exe, tmp):
    argv = [exe]
    for f, c in ARGS:
        argv += [os.path.join(tmp, f), c]
    return subprocess.run(argv, capture_output=True, text=True, check=True).stdout


def test_load_series_matches_reference(tmp_path):
    lib = os.path.join(PKG, "libtsdiscord_b200.so")
    if not os.path.exists(lib):
        pytest.skip("library not built")
    if not (os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/include")):
        pytest.skip("reference library not built here")
    for name, text in CASES.items():
        (tmp_path / name).write_text(text)
    ours, ref = str(tmp_path / "ours"), str(tmp_path / "ref")
    build(tmp_path, PKG, "tsdiscord_b200", os.path.join(ROOT, "include"), ours)
    build(tmp_path, os.path.dirname(REF_SO), "tsdref", "/root/reference/proj/include", ref)
    a, b = run(ours, str(tmp_path)), run(ref, str(tmp_path))
    assert a == b
    assert a.count("ok ") >= 6


def test_load_series_large_parallel(tmp_path):
    # > 65536 lines: the parallel path; values and the first error by line number
    lib = os.path.join(PKG, "libtsdiscord_b200.so")
    if not os.path.exists(lib):
        pytest.skip("library not built")
    import numpy as np
    x = np.random.default_rng(5).normal(size=300_000).cumsum()
    lines = [repr(float(v)) for v in x]
    (tmp_path / "big.txt").write_text("\n".join(lines) + "\n")
    bad = list(lines)
    bad[200_000] = "oops"
    bad[250_000] = "worse"
    (tmp_path / "bad.txt").write_text("\n".join(bad) + "\n")
    exe = str(tmp_path / "ours")
    build(tmp_path, PKG, "tsdiscord_b200", os.path.join(ROOT, "include"), exe)
    out = subprocess.run([exe, str(tmp_path / "big.txt"), "-", str(tmp_path / "bad.txt"), "-"],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    vals = np.array([float(v) for v in out[0].split()[2:]])
    assert int(out[0].split()[1]) == len(x) and np.array_equal(vals, x)
    assert out[1] == "runtime_error: line 200001: non-numeric value 'oops'"
