import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    p = os.path.join(GOLDEN, name)
    if not os.path.exists(p):
        pytest.skip(f"golden fixture {name} not generated")
    with open(p) as f:
        return json.load(f)


def hexf(s):
    return float.fromhex(s)


def series_of(inp):
    """Regenerates a fixture's input series (the library's generators)."""
    import hashlib

    from paper_2304_01660_b200.datasets import make_series
    x = make_series(inp)
    if "sha256" in inp:  # generators with transcendental math: the input itself is pinned
        assert hashlib.sha256(x.tobytes()).hexdigest() == inp["sha256"], "fixture input differs"
    return x


@pytest.fixture(scope="session")
def oracle():
    from oracle.refbind import Oracle
    try:
        return Oracle()
    except FileNotFoundError:
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
        return Oracle()


@pytest.fixture(scope="session")
def engine():
    import torch  # noqa: F401  (only to probe the device cheaply)
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_01660_b200 import Engine
    return Engine(0)
