"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Ref``    -> ``oracle/_ref/libtsdref.so``: the UNMODIFIED reference library
                (``/root/reference/proj/src``) built by ``oracle/Makefile`` plus the
                extern "C" shim ``oracle/ref_shim.cpp``.
* ``Oracle`` -> ``oracle/liboracle.so``: the plain-C restatement ``oracle/oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtsdref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

REC_DTYPE = np.dtype([("index", np.int64), ("nn_dist_sq", np.float64), ("nn_dist", np.float64)])

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64 = C.c_int64


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _as_series(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


class _Common:
    prefix = ""

    def _fn(self, name, restype, argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        f.argtypes = argtypes
        return f

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(rc, getattr(self.lib, self.prefix + "last_error")().decode())

    def _bind_common(self):
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p
        self._gen = self._fn("gen_randomwalk", C.c_int, [_i64, C.c_uint64, _dp])
        self._init = self._fn("init_stats", C.c_int, [_dp, _i64, _i64, _dp, _dp])
        self._adv = self._fn("advance_stats", C.c_int, [_dp, _i64, _i64, _i64, _dp, _dp])
        self._bf = self._fn("brute_force_nn", C.c_int, [_dp, _i64, _i64, _dp])
        self._merlin = self._fn(
            "merlin", C.c_int,
            [_dp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, C.c_int, _ip, C.c_void_p, _dp, _ip, _u8])

    def gen_randomwalk(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self._check(self._gen(n, seed, out))
        return out

    def init_stats(self, x, m: int):
        x = _as_series(x)
        N = len(x) - m + 1
        mu, sg = np.empty(max(N, 1)), np.empty(max(N, 1))
        self._check(self._init(x, len(x), m, mu, sg))
        return mu[:N], sg[:N]

    def advance_stats(self, x, m0: int, m1: int):
        """init_stats(m0) advanced (m1-m0) times with the Eq. 7-8 recurrence."""
        x = _as_series(x)
        N = len(x) - m1 + 1
        mu, sg = np.empty(max(len(x) - m0 + 1, 1)), np.empty(max(len(x) - m0 + 1, 1))
        self._check(self._adv(x, len(x), m0, m1, mu, sg))
        return mu[:N], sg[:N]

    def brute_force_nn(self, x, m: int) -> np.ndarray:
        x = _as_series(x)
        out = np.empty(len(x) - m + 1)
        self._check(self._bf(x, len(x), m, out))
        return out

    def merlin(self, x, min_len, max_len, top_k=1, seglen=512, workers=1, max_retries=100,
               reuse_stats=True):
        """Returns dict(counts, recs[L, top_k], final_r, retries, failed)."""
        x = _as_series(x)
        L = max_len - min_len + 1
        counts = np.zeros(max(L, 1), np.int64)
        recs = np.zeros((max(L, 1), top_k), REC_DTYPE)
        final_r = np.zeros(max(L, 1))
        retries = np.zeros(max(L, 1), np.int64)
        failed = np.zeros(max(L, 1), np.uint8)
        self._check(self._merlin(x, len(x), min_len, max_len, top_k, seglen, workers, max_retries,
                                 1 if reuse_stats else 0, counts, recs.ctypes.data, final_r,
                                 retries, failed))
        return dict(counts=counts[:L], recs=recs[:L], final_r=final_r[:L], retries=retries[:L],
                    failed=failed[:L])


class Ref(_Common):
    """The reference library itself (needs oracle/_ref/libtsdref.so)."""

    prefix = "tsdref_"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(path)
        self._bind_common()
        self._pardrag = self._fn("pardrag", C.c_int,
                                 [_dp, _i64, _i64, C.c_double, _i64, _i64, C.c_void_p, _i64,
                                  C.POINTER(_i64)])
        self._csv = self._fn("merlin_csv", _i64, [_dp, _i64, _i64, _i64, _i64, _i64, _i64,
                                                  C.c_char_p, _i64])
        self._hm = self._fn("heatmap", _i64, [C.c_char_p, _i64, _i64, C.c_int, C.c_char_p, _i64])

    def heatmap(self, csv: str, n: int, k: int = 10, which: int = 0) -> bytes:
        """The reference CLI's heatmap outputs: 0 heatmap CSV, 1 PGM, 2 ranking CSV."""
        size = self._hm(csv.encode(), n, k, which, None, 0)
        if size < 0:
            raise CheckerError(3, self.lib.tsdref_last_error().decode())
        buf = C.create_string_buffer(size + 1)
        self._hm(csv.encode(), n, k, which, buf, size)
        return buf.raw[:size]

    def pardrag(self, x, m: int, r_sq: float, seglen: int, workers: int = 1) -> np.ndarray:
        x = _as_series(x)
        cap = len(x)
        recs = np.zeros(cap, REC_DTYPE)
        cnt = _i64(0)
        self._check(self._pardrag(x, len(x), m, r_sq, seglen, workers, recs.ctypes.data, cap,
                                  C.byref(cnt)))
        return recs[: cnt.value].copy()

    def merlin_csv(self, x, min_len, max_len, top_k=1, seglen=512, workers=1) -> str:
        x = _as_series(x)
        size = self._csv(x, len(x), min_len, max_len, top_k, seglen, workers, None, 0)
        if size < 0:
            raise CheckerError(3, self.lib.tsdref_last_error().decode())
        buf = C.create_string_buffer(size + 1)
        self._csv(x, len(x), min_len, max_len, top_k, seglen, workers, buf, size)
        return buf.raw[:size].decode()


class Oracle(_Common):
    """The plain-C restatement (oracle/oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self._bind_common()
        self._range = self._fn("range_discords", _i64,
                               [_dp, _i64, _i64, C.c_double, C.c_void_p, _i64])
        self._layout = self._fn("compute_layout", C.c_int,
                                [_i64, _i64, _i64, C.POINTER(_i64 * 4)])
        self._thr = self._fn("next_threshold", C.c_int,
                             [_dp, _i64, C.c_int, _i64, C.c_double, C.c_int,
                              C.POINTER(C.c_double)])
        self._pair = self._fn("ref_sq_dist", C.c_double, [_dp, _i64, _i64, _i64, _i64])

    def range_discords(self, x, m: int, r_sq: float) -> np.ndarray:
        """{i : nn(i) >= r_sq} with exact nn, sorted (nn desc, index asc)."""
        x = _as_series(x)
        cap = len(x)
        recs = np.zeros(cap, REC_DTYPE)
        cnt = self._range(x, len(x), m, r_sq, recs.ctypes.data, cap)
        if cnt < 0:
            self._check(int(-cnt))
        return recs[:cnt].copy()

    def compute_layout(self, n, m, seglen):
        out = (_i64 * 4)()
        self._check(self._layout(n, m, seglen, C.byref(out)))
        return dict(seglen=out[0], seg_n=out[1], num_seg=out[2], pad=out[3])

    def next_threshold(self, history, phase: int, min_len: int, last_r: float, failed: bool):
        h = _as_series(history) if len(history) else np.zeros(1)
        r = C.c_double(0)
        self._check(self._thr(h, len(history), phase, min_len, last_r, 1 if failed else 0,
                              C.byref(r)))
        return r.value

    def ref_sq_dist(self, x, m, i, j) -> float:
        """reference_sq_dist (1-based i, j)."""
        x = _as_series(x)
        return self._pair(x, len(x), m, i, j)
