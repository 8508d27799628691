"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/tsdiscord_b200.h declares, and its host-side arithmetic
(layout, threshold schedule, generator) equals the reference's."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_2304_01660_b200 as P


def test_header_declares_exactly_the_exports():
    hdr = open(os.path.join(ROOT, "include", "tsdiscord_b200.h")).read()
    declared = set(re.findall(r"\b(tsd_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(P.EXPORTS)


def test_library_exports_every_symbol():
    P.load_library()
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [s for s in P.EXPORTS if s not in syms]
    assert not missing, missing


def test_library_carries_sm100a_code():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_compute_layout_known_answers():
    # reference tests/types_test.cpp:9-25
    assert P.compute_layout(100, 10, 32) == dict(seglen=32, seg_n=23, num_seg=4, pad=10)
    assert P.compute_layout(101, 10, 32)["pad"] == 9
    assert P.compute_layout(100, 10, 10) == dict(seglen=10, seg_n=1, num_seg=91, pad=9)
    for bad in [(100, 2, 32), (100, 99, 99), (100, 10, 9), (100, 10, 101)]:
        with pytest.raises(ValueError):
            P.compute_layout(*bad)


def test_compute_layout_random_against_oracle(oracle):
    rng = np.random.default_rng(88)
    for _ in range(2000):  # acceptance criterion 8 (padding formula)
        n = int(rng.integers(50, 5000))
        m = int(rng.integers(3, max(4, n // 3)))
        if m > n - 2:
            continue
        seglen = int(m + rng.integers(0, n - m + 1))
        assert P.compute_layout(n, m, seglen) == oracle.compute_layout(n, m, seglen)


def test_threshold_schedule_constants():
    # reference tests/merlin_test.cpp:11-45 and acceptance criterion 6
    assert P.next_threshold([], P.FIRST, 64, 0.0, False) == 16.0
    assert P.next_threshold([], P.FIRST, 64, 16.0, True) == 8.0
    assert abs(P.next_threshold([10.0], P.WARMUP, 8, 0.0, False) - 9.9) < 1e-12
    assert abs(P.next_threshold([10.0], P.WARMUP, 8, 9.9, True) - 9.9 * 0.99) < 1e-12
    st = [3.5, 4.5, 4.0, 4.5, 3.5]
    sd = float(np.std(st))
    assert abs(P.next_threshold(st, P.STEADY, 8, 0.0, False) - (4.0 - 2 * sd)) < 1e-12
    assert abs(P.next_threshold(st, P.STEADY, 8, 3.0, True) - (3.0 - sd)) < 1e-12
    assert abs(P.next_threshold([3.0] * 5, P.STEADY, 8, 3.0, True) - 2.97) < 1e-12
    assert abs(P.next_threshold([0.1, 10.0, 0.1, 10.0, 0.2], P.STEADY, 8, 0.0, False) - 0.002) < 1e-15
    with pytest.raises(P.LogicError):  # merlin.cpp:19
        P.next_threshold([1.0, 2.0], P.STEADY, 8, 0.0, False)


def test_schedule_bitexact_vs_oracle(oracle):
    rng = np.random.default_rng(6)
    for _ in range(500):
        h = list(rng.uniform(0.5, 20.0, size=int(rng.integers(5, 12))))
        ph = int(rng.integers(0, 3))
        last = float(rng.uniform(0.1, 20))
        f = bool(rng.integers(0, 2))
        assert P.next_threshold(h, ph, 17, last, f) == oracle.next_threshold(h, ph, 17, last, f)


def test_generator_matches_reference():
    for e in load_golden("small.json")["randomwalk"]:
        x = P.gen_randomwalk(e["n"], e["seed"])
        assert [v.hex() for v in x[:8].tolist()] == e["head"]
        assert x[-1].hex() == e["last"]
    with pytest.raises(ValueError):
        P.gen_randomwalk(2, 1)


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        P.Engine(0)


def test_cpp_dropin_exports_reference_declarations():
    # every function the reference headers declare (proj/include/tsdiscord/*.hpp)
    # is defined by libtsdiscord_b200.so, so a reference caller relinks unchanged
    P.load_library()
    out = subprocess.run(["nm", "-DC", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    for sym in ["tsdiscord::znormalize(", "tsdiscord::sq_ed(", "tsdiscord::sq_ednorm_from_dot(",
                "tsdiscord::early_abandon_sq_ed(", "tsdiscord::dot_products_block(",
                "tsdiscord::update_dot_col(", "tsdiscord::drag_select(", "tsdiscord::drag_refine(",
                "tsdiscord::drag(", "tsdiscord::brute_force_nn(", "tsdiscord::brute_force_topk(",
                "tsdiscord::par_select(", "tsdiscord::par_refine(", "tsdiscord::pardrag(",
                "tsdiscord::SelectionState::SelectionState(", "tsdiscord::SelectionState::conjoin(",
                "tsdiscord::SelectionState::lower_nn_dist_sq(", "tsdiscord::merlin(",
                "tsdiscord::merlin_full(", "tsdiscord::next_threshold(", "tsdiscord::init_stats(",
                "tsdiscord::advance_stats(", "tsdiscord::compute_layout(", "tsdiscord::build_heatmap(",
                "tsdiscord::rank_discords(", "tsdiscord::load_series(", "tsdiscord::gen_randomwalk(",
                "tsdiscord::write_discords_csv(", "tsdiscord::read_discords_csv("]:
        assert sym in out, sym


def test_reference_acceptance_gate_links():
    # built by build() from the unchanged reference test (tests/cpp/Makefile)
    gate = os.path.join(ROOT, "tests", "cpp", "_ref", "acceptance")
    if not os.path.exists(gate):
        pytest.skip("acceptance gate not built (needs /root/reference)")
    out = subprocess.run(["ldd", gate], capture_output=True, text=True).stdout
    assert "libtsdiscord_b200.so" in out and "not found" not in out
