"""Synthetic inputs for the BASELINE configurations.

* random walk: ``gen_randomwalk`` (the reference's generator, src/io.cpp:110-119,
  in the C-ABI so it is bit-identical to the reference).
* ECG-like (BASELINE config 3; the reference has no generator):
  a quasi-periodic beat of Gaussian P/Q/R/S/T bumps (~250 samples per beat),
  +-2% period jitter, +-5% amplitude jitter, additive Gaussian noise sigma=0.05,
  and K injected anomalies (missing QRS, doubled beat, amplitude x2, flat-line
  shorter than one beat).  Noise is added everywhere, so no stretch is exactly
  constant or exactly periodic.  Deterministic for a given seed (numpy PCG64).
"""
from __future__ import annotations

import math

import numpy as np

# (centre as a fraction of the beat, width in samples, amplitude) of P, Q, R, S, T
_WAVES = ((0.18, 9.0, 0.15), (0.36, 3.5, -0.12), (0.40, 3.0, 1.0), (0.44, 3.5, -0.25), (0.68, 16.0, 0.30))


def _beat(length: int, amp: float, qrs: bool = True) -> np.ndarray:
    # scalar libm exp (math.exp), not numpy's SIMD exp: numpy picks its exp kernel
    # by the host CPU's features, and the fixture must regenerate bit-identically on
    # the GPU box's host
    out = [0.0] * length
    for k, (c, w, a) in enumerate(_WAVES):
        if not qrs and k in (1, 2, 3):
            continue
        ctr, aa = c * length, a * amp
        for i in range(length):
            z = (i - ctr) / w
            out[i] += aa * math.exp(-0.5 * z * z)
    return np.asarray(out, dtype=np.float64)


def gen_ecg_like(n: int, seed: int, period: int = 250, n_anomalies: int = 10) -> np.ndarray:
    rng = np.random.default_rng(seed)
    beats = []
    total = 0
    while total < n + 2 * period:
        length = int(round(period * (1.0 + rng.uniform(-0.02, 0.02))))
        beats.append(length)
        total += length
    nb = len(beats)
    kinds = ["missing_qrs", "double", "amp2", "flat"]
    anomalous = {}
    if n_anomalies > 0:
        picks = rng.choice(np.arange(2, nb - 2), size=min(n_anomalies, nb - 4), replace=False)
        for i, b in enumerate(sorted(picks.tolist())):
            anomalous[b] = kinds[i % len(kinds)]
    parts = []
    for b, length in enumerate(beats):
        amp = 1.0 + rng.uniform(-0.05, 0.05)
        kind = anomalous.get(b)
        if kind == "missing_qrs":
            parts.append(_beat(length, amp, qrs=False))
        elif kind == "double":
            h = length // 2
            parts.append(np.concatenate([_beat(h, amp), _beat(length - h, amp)]))
        elif kind == "amp2":
            parts.append(_beat(length, 2.0 * amp))
        elif kind == "flat":
            parts.append(np.zeros(length))
        else:
            parts.append(_beat(length, amp))
    x = np.concatenate(parts)[:n]
    x = x + rng.normal(0.0, 0.05, size=n)
    return np.ascontiguousarray(x, dtype=np.float64)


def make_series(spec: dict) -> np.ndarray:
    """Builds the input described by a fixture / bench spec {"gen": ..., "n": ..., "seed": ...}."""
    if spec["gen"] == "randomwalk":
        from . import gen_randomwalk

        x = gen_randomwalk(spec["n"], spec["seed"])
        return x + spec["offset"] if spec.get("offset") else x
    if spec["gen"] == "ecg":
        return gen_ecg_like(spec["n"], spec["seed"])
    raise ValueError(f"unknown generator {spec['gen']}")
