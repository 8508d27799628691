"""paper_2304_01660_b200 — B200-native PALMAD (arXiv 2304.01660) discord discovery.

Python binding of ``libtsdiscord_b200.so`` (C-ABI in ``include/tsdiscord_b200.h``).
The names mirror the reference's C++ API (``/root/reference/proj/include/tsdiscord``):
``merlin``, ``merlin_full``, ``pardrag``, ``init_stats``, ``advance_stats``,
``compute_layout``, ``next_threshold``, ``brute_force_nn``, ``gen_randomwalk``, with the
same argument meaning and the same exception kinds (``ValueError`` for the
reference's ``std::invalid_argument``, ``LogicError`` for ``std::logic_error``,
``RuntimeError`` otherwise).  Every compute call runs on the GPU; a missing
library or device raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSD_LIB") or os.path.join(HERE, "libtsdiscord_b200.so")  # TSD_LIB: A/B experiments

TSD_OK, TSD_EINVAL, TSD_ELOGIC, TSD_ERUNTIME, TSD_ECUDA = range(5)

RECORD_DTYPE = np.dtype([("index", np.int64), ("nn_dist_sq", np.float64), ("nn_dist", np.float64)])

# Every symbol include/tsdiscord_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "tsd_ctx_create", "tsd_ctx_destroy", "tsd_last_error", "tsd_create_error",
    "tsd_nccl_unique_id", "tsd_ctx_join", "tsd_series_set", "tsd_series_len",
    "tsd_init_stats", "tsd_advance_stats", "tsd_compute_layout", "tsd_next_threshold",
    "tsd_pardrag", "tsd_merlin", "tsd_brute_force_nn", "tsd_gen_randomwalk",
    "tsd_get_counters", "tsd_reset_counters", "tsd_set_param", "tsd_fp32_peak_probe",
    "tsd_heatmap_build", "tsd_heatmap_set", "tsd_heatmap_rank",
    "tsd_group_create", "tsd_group_destroy", "tsd_group_last_error", "tsd_group_size", "tsd_group_ctx",
    "tsd_group_series_set", "tsd_group_merlin", "tsd_group_pardrag", "tsd_matrix_profile_fp64",
    "tsd_ipc_export", "tsd_ipc_join", "tsd_par_select", "tsd_par_refine", "tsd_stats_walk",
    "tsd_seed_rows", "tsd_tile_plan",
)


class LogicError(RuntimeError):
    """std::logic_error of the reference (e.g. merlin.cpp:19 window too short)."""


RANKED_DTYPE = np.dtype([("index", np.int64), ("length", np.int64), ("score", np.float64)])


class _Opts(C.Structure):
    _fields_ = [("top_k", C.c_int64), ("seglen", C.c_int64), ("workers", C.c_int64),
                ("max_retries", C.c_int64), ("reuse_stats", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [("cells", C.c_uint64), ("cells_eval", C.c_uint64), ("seed_dots", C.c_uint64),
                ("seed_flops", C.c_uint64), ("rechecks", C.c_uint64), ("exact_pairs", C.c_uint64),
                ("pardrag_calls", C.c_uint64), ("scan_launches", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("host_syncs", C.c_uint64),
                ("scan_ms", C.c_double), ("dense_ms", C.c_double), ("sparse_ms", C.c_double),
                ("collect_ms", C.c_double), ("total_ms", C.c_double),
                ("host_wall_ms", C.c_double), ("host_wait_ms", C.c_double),
                ("heatmap_ms", C.c_double), ("fallbacks", C.c_uint64),
                ("wit_tests", C.c_uint64), ("wit_kills", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_lib = None


def load_library(path: str = LIB_PATH):
    """Loads (once) and binds the C-ABI.  Raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2304_01660_b200.build`")
    L = C.CDLL(path)

    def f(name, res, args):
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args

    vp = C.c_void_p
    f("tsd_ctx_create", C.c_int, [C.c_int, C.POINTER(vp)])
    f("tsd_ctx_destroy", None, [vp])
    f("tsd_last_error", C.c_char_p, [vp])
    f("tsd_create_error", C.c_char_p, [])
    f("tsd_nccl_unique_id", C.c_int, [C.c_char_p])
    f("tsd_ctx_join", C.c_int, [vp, C.c_int, C.c_int, C.c_char_p])
    f("tsd_series_set", C.c_int, [vp, _dp, _i64])
    f("tsd_series_len", _i64, [vp])
    f("tsd_init_stats", C.c_int, [vp, _i64, _dp, _dp])
    f("tsd_advance_stats", C.c_int, [vp, _i64, _dp, _dp, _dp, _dp])
    f("tsd_compute_layout", C.c_int, [_i64, _i64, _i64, _ip])
    f("tsd_next_threshold", C.c_int, [_dp, _i64, C.c_int, _i64, C.c_double, C.c_int,
                                      C.POINTER(C.c_double)])
    f("tsd_pardrag", C.c_int, [vp, _i64, C.c_double, _i64, vp, vp, vp, _i64, C.POINTER(_i64)])
    f("tsd_par_select", C.c_int, [vp, _i64, C.c_double, _i64, vp, vp, _u8, _dp])
    f("tsd_par_refine", C.c_int, [vp, _i64, C.c_double, _i64, vp, vp, _u8, vp, _i64, C.POINTER(_i64)])
    f("tsd_stats_walk", C.c_int, [vp, _i64, _i64, C.c_int, _dp, _dp])
    f("tsd_tile_plan", C.c_int, [C.c_int, _i64, _i64, _i64, _i64, _i64, _i64, vp, _i64, C.c_int, C.c_int,
                                 vp, _i64, C.POINTER(_i64)])
    f("tsd_seed_rows", C.c_int, [vp, vp, _i64, _ip])
    f("tsd_merlin", C.c_int, [vp, _i64, _i64, C.POINTER(_Opts), _ip, vp, _dp, _ip, _u8])
    f("tsd_brute_force_nn", C.c_int, [vp, _i64, _dp])
    f("tsd_matrix_profile_fp64", C.c_int, [vp, _i64, _dp])
    f("tsd_ipc_export", C.c_int, [vp, _i64, C.c_char_p])
    f("tsd_ipc_join", C.c_int, [vp, C.c_int, C.c_int, C.c_char_p, C.c_char_p])
    f("tsd_gen_randomwalk", C.c_int, [_i64, C.c_uint64, _dp])
    f("tsd_get_counters", C.c_int, [vp, C.POINTER(Counters)])
    f("tsd_reset_counters", C.c_int, [vp])
    f("tsd_set_param", C.c_int, [vp, C.c_char_p, C.c_double])
    f("tsd_fp32_peak_probe", C.c_int, [C.c_int, C.POINTER(C.c_double)])
    f("tsd_group_create", C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)])
    f("tsd_group_destroy", None, [vp])
    f("tsd_group_last_error", C.c_char_p, [vp])
    f("tsd_group_ctx", vp, [vp, C.c_int])
    f("tsd_group_series_set", C.c_int, [vp, _dp, _i64])
    f("tsd_group_merlin", C.c_int, [vp, _i64, _i64, C.POINTER(_Opts), _ip, vp, _dp, _ip, _u8])
    f("tsd_group_pardrag", C.c_int, [vp, _i64, C.c_double, _i64, vp, _i64, C.POINTER(_i64)])
    f("tsd_heatmap_build", C.c_int, [vp, _i64, _i64, _i64, _ip, vp, _i64, vp])
    f("tsd_heatmap_set", C.c_int, [vp, _i64, _i64, _i64, _dp])
    f("tsd_heatmap_rank", C.c_int, [vp, _i64, vp, C.POINTER(_i64)])
    _lib = L
    return L


def _raise(code: int, msg: str):
    if code == TSD_EINVAL:
        raise ValueError(msg)
    if code == TSD_ELOGIC:
        raise LogicError(msg)
    raise RuntimeError(msg)


def _host_check(rc):
    if rc != TSD_OK:
        _raise(rc, (load_library().tsd_last_error(None) or b"").decode())


# ---------------------------------------------------------------------------
# host arithmetic (bit-exact restatements, no device needed)
def compute_layout(n: int, m: int, seglen: int) -> dict:
    """src/types.cpp:26-39 -> {seglen, seg_n, num_seg, pad}; ValueError on bad input."""
    out = np.zeros(4, np.int64)
    _host_check(load_library().tsd_compute_layout(n, m, seglen, out))
    return dict(seglen=int(out[0]), seg_n=int(out[1]), num_seg=int(out[2]), pad=int(out[3]))


FIRST, WARMUP, STEADY = 0, 1, 2


def next_threshold(history, phase: int, min_len: int, last_r: float, failed: bool) -> float:
    """src/merlin.cpp:35-55 (phase 0 first, 1 warmup, 2 steady)."""
    h = np.ascontiguousarray(history, dtype=np.float64) if len(history) else np.zeros(1)
    r = C.c_double(0.0)
    _host_check(load_library().tsd_next_threshold(h, len(history), phase, min_len, last_r,
                                                   1 if failed else 0, C.byref(r)))
    return r.value


TILE_SPACES = {"seed": 0, "blocks": 1, "band": 2, "full": 3}


def tile_plan(space: str, N: int, m: int, rank: int = 0, world: int = 1, L: int = 512, kA: int = 0,
              nb: int = 1, K0: int = 0, groups=None) -> np.ndarray:
    """Tiles {r0, rows, k0, dir, seed} rank `rank` of `world` scans in one launch
    of the given tile space (the kernels' own decoder; host only, no GPU)."""
    L_ = load_library()
    g = None
    G = 0
    if groups is not None:
        g = np.ascontiguousarray(np.asarray(groups, dtype=np.int32).reshape(-1, 2))
        G = len(g)
    cnt = _i64(0)
    _host_check(L_.tsd_tile_plan(TILE_SPACES[space], N, m, L, kA, nb, K0,
                                 g.ctypes.data if g is not None else None, G, rank, world, None, 0,
                                 C.byref(cnt)))
    out = np.zeros((max(cnt.value, 1), 5), np.int32)
    _host_check(L_.tsd_tile_plan(TILE_SPACES[space], N, m, L, kA, nb, K0,
                                 g.ctypes.data if g is not None else None, G, rank, world,
                                 out.ctypes.data, cnt.value, C.byref(cnt)))
    return out[: cnt.value]


def fp32_peak_tflops(device: int = 0) -> float:
    """Measured FP32 FFMA peak of the device (diagnostic microbenchmark)."""
    v = C.c_double(0.0)
    _host_check(load_library().tsd_fp32_peak_probe(device, C.byref(v)))
    return v.value


def gen_randomwalk(n: int, seed: int) -> np.ndarray:
    """src/io.cpp:110-119: x1 = 0, x_{i+1} = x_i + N(0,1) (libstdc++ mt19937_64)."""
    out = np.empty(max(n, 1), np.float64)
    _host_check(load_library().tsd_gen_randomwalk(n, seed, out))
    return out[:n]


# ---------------------------------------------------------------------------
@dataclass
class MerlinReport:
    """merlin.hpp:40-44; per_length maps m -> structured array of records."""
    min_len: int
    max_len: int
    per_length: dict = field(default_factory=dict)
    failed_lengths: list = field(default_factory=list)
    final_r: np.ndarray = None
    retries: np.ndarray = None
    device_ms: float = 0.0


class Engine:
    """One GPU context (device, stream, resident series, scan state)."""

    def __init__(self, device: int = 0):
        L = load_library()
        self._L = L
        h = C.c_void_p()
        rc = L.tsd_ctx_create(device, C.byref(h))
        if rc != TSD_OK:
            _raise(rc, (L.tsd_create_error() or b"").decode())
        self._h = h
        self._series = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.tsd_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != TSD_OK:
            _raise(rc, (self._L.tsd_last_error(self._h) or b"").decode())

    # -- multi-GPU --------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _host_check(load_library().tsd_nccl_unique_id(buf))
        return buf.raw

    def ipc_export(self, rows: int) -> bytes:
        """Cross-process ranks, step 1: allocate the shared arrays (rows >= series
        length) and return this rank's 320 bytes of CUDA IPC handles."""
        buf = C.create_string_buffer(320)
        self._check(self._L.tsd_ipc_export(self._h, rows, buf))
        return buf.raw

    def ipc_join(self, rank: int, world: int, handles: list, shm_name: str):
        """Step 2: join with every rank's handles (rank order); rank 0 first."""
        blob = b"".join(handles)
        assert len(blob) == 320 * world
        self._check(self._L.tsd_ipc_join(self._h, rank, world, blob, shm_name.encode()))

    def join(self, rank: int, world: int, nccl_id: bytes | None = None):
        idb = C.create_string_buffer(nccl_id or b"\0" * 128, 128)
        self._check(self._L.tsd_ctx_join(self._h, rank, world, idb))

    # -- series / stats -----------------------------------------------------
    def set_series(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self._L.tsd_series_set(self._h, x, len(x)))
        self._series = x

    @property
    def n(self) -> int:
        return int(self._L.tsd_series_len(self._h))

    def init_stats(self, m: int):
        N = max(self.n - m + 1, 1)
        mu, sg = np.empty(N), np.empty(N)
        self._check(self._L.tsd_init_stats(self._h, m, mu, sg))
        return mu, sg

    def advance_stats(self, m: int, mu, sigma):
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        N = max(self.n - m, 1)
        mo, so = np.empty(N), np.empty(N)
        self._check(self._L.tsd_advance_stats(self._h, m, mu, sigma, mo, so))
        return mo, so

    # -- scans --------------------------------------------------------------
    def pardrag(self, m: int, r_sq: float, seglen: int, stats=None) -> np.ndarray:
        N = max(self.n - m + 1, 1)
        out = np.zeros(N, RECORD_DTYPE)
        cnt = _i64(0)
        mu = sg = None
        if stats is not None:
            mu = np.ascontiguousarray(stats[0], dtype=np.float64)
            sg = np.ascontiguousarray(stats[1], dtype=np.float64)
        self._check(self._L.tsd_pardrag(
            self._h, m, float(r_sq), seglen,
            mu.ctypes.data if mu is not None else None,
            sg.ctypes.data if sg is not None else None,
            out.ctypes.data, N, C.byref(cnt)))
        return out[: cnt.value].copy()

    def par_select(self, m: int, r_sq: float, seglen: int):
        """(cand u8[N], nn f64[N]) of the selection phase (pardrag.hpp:71-73)."""
        N = max(self.n - m + 1, 1)
        cand, nn = np.zeros(N, np.uint8), np.empty(N)
        self._check(self._L.tsd_par_select(self._h, m, float(r_sq), seglen, None, None, cand, nn))
        return cand, nn

    def par_refine(self, m: int, r_sq: float, seglen: int, cand) -> np.ndarray:
        N = max(self.n - m + 1, 1)
        cand = np.ascontiguousarray(cand, dtype=np.uint8)
        out = np.zeros(N, RECORD_DTYPE)
        cnt = _i64(0)
        self._check(self._L.tsd_par_refine(self._h, m, float(r_sq), seglen, None, None, cand,
                                           out.ctypes.data, N, C.byref(cnt)))
        return out[: cnt.value].copy()

    def stats_walk(self, m0: int, m1: int, fused: bool = True):
        """mu/sigma of length m1 after MERLIN's length steps from m0 (the fused
        k_next_length path by default)."""
        N = max(self.n - m1 + 1, 1)
        mu, sg = np.empty(N), np.empty(N)
        self._check(self._L.tsd_stats_walk(self._h, m0, m1, 1 if fused else 0, mu, sg))
        return mu, sg

    def seed_rows(self):
        """(info {m, L, kA, nb}, rows f64[nb, 1152]) of the resident band-0 seed rows."""
        info = np.zeros(4, np.int64)
        self._check(self._L.tsd_seed_rows(self._h, None, 0, info))
        rows = np.empty((int(info[3]), 1152))
        if info[3] > 0:
            self._check(self._L.tsd_seed_rows(self._h, rows.ctypes.data, rows.size, info))
        return info, rows

    def brute_force_nn(self, m: int) -> np.ndarray:
        out = np.empty(max(self.n - m + 1, 1))
        self._check(self._L.tsd_brute_force_nn(self._h, m, out))
        return out

    def matrix_profile_fp64(self, m: int) -> np.ndarray:
        """Independent FP64 matrix profile (checker; ~1e-10 relative to brute_force_nn)."""
        out = np.empty(max(self.n - m + 1, 1))
        self._check(self._L.tsd_matrix_profile_fp64(self._h, m, out))
        return out

    def merlin_full(self, min_len: int, max_len: int, top_k: int = 1, seglen: int = 512,
                    workers: int = 1, max_retries: int = 100, reuse_stats: bool = True) -> MerlinReport:
        Ln = max(max_len - min_len + 1, 1)
        k = max(top_k, 1)
        counts = np.zeros(Ln, np.int64)
        recs = np.zeros((Ln, k), RECORD_DTYPE)
        final_r = np.zeros(Ln)
        retries = np.zeros(Ln, np.int64)
        failed = np.zeros(Ln, np.uint8)
        o = _Opts(top_k, seglen, workers, max_retries, 1 if reuse_stats else 0)
        self._check(self._L.tsd_merlin(self._h, min_len, max_len, C.byref(o), counts,
                                       recs.ctypes.data, final_r, retries, failed))
        rep = MerlinReport(min_len, max_len, final_r=final_r[: max_len - min_len + 1],
                           retries=retries[: max_len - min_len + 1])
        for i in range(max_len - min_len + 1):
            m = min_len + i
            if failed[i]:
                rep.failed_lengths.append(m)
            else:
                rep.per_length[m] = recs[i][: counts[i]].copy()
        rep.device_ms = self.counters()["total_ms"]
        return rep

    # -- heatmap / ranking (heatmap.hpp) ---------------------------------------
    def heatmap(self, per_length: dict, n: int, min_len: int | None = None, max_len: int | None = None,
                scores: bool = False):
        """build_heatmap (heatmap.cpp:18-31) on the device; returns the
        (rows, cols) score matrix when `scores`, else None (it stays resident
        for heatmap_rank)."""
        lens = sorted(per_length)
        if min_len is None:
            min_len = lens[0] if lens else 0
        if max_len is None:
            max_len = lens[-1] if lens else -1
        ls, rs = [], []
        for m in lens:
            for r in per_length[m]:
                ls.append(m)
                rs.append((int(r["index"]), float(r["nn_dist_sq"]), float(r["nn_dist"])))
        recs = np.array(rs, dtype=RECORD_DTYPE) if rs else np.zeros(1, RECORD_DTYPE)
        lens_a = np.array(ls if ls else [0], dtype=np.int64)
        out = None
        if scores and min_len >= 3 and max_len >= min_len and n > max_len:
            out = np.empty((max_len - min_len + 1, n - min_len))
        self._check(self._L.tsd_heatmap_build(self._h, min_len, max_len, n, lens_a, recs.ctypes.data, len(rs),
                                              out.ctypes.data if out is not None else None))
        return out

    def heatmap_set(self, scores, min_len: int, max_len: int, n: int):
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        self._check(self._L.tsd_heatmap_set(self._h, min_len, max_len, n, sc.ravel()))

    def heatmap_rank(self, k: int) -> np.ndarray:
        """rank_discords (heatmap.cpp:33-57): per-column max on the device."""
        cap = max(int(k), 1)
        out = np.zeros(cap, RANKED_DTYPE)
        cnt = C.c_int64(0)
        self._check(self._L.tsd_heatmap_rank(self._h, k, out.ctypes.data, C.byref(cnt)))
        return out[: cnt.value].copy()

    # -- accounting / knobs ---------------------------------------------------
    def counters(self) -> dict:
        c = Counters()
        self._check(self._L.tsd_get_counters(self._h, C.byref(c)))
        return c.as_dict()

    def reset_counters(self):
        self._check(self._L.tsd_reset_counters(self._h))

    def set_param(self, key: str, value: float):
        self._check(self._L.tsd_set_param(self._h, key.encode(), float(value)))


class Group:
    """In-process rank group (tsd_group_*): rank r runs on devices[r] (repeats
    allowed), tiles are dealt cyclically over the ranks and reductions go
    through peer memory.  Same results as Engine, bit for bit."""

    def __init__(self, devices):
        self._L = load_library()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        rc = self._L.tsd_group_create(devs, len(devices), C.byref(h))
        if rc != TSD_OK:
            _raise(rc, (self._L.tsd_create_error() or b"").decode())
        self._h = h
        self.size = len(devices)
        self.n = 0

    def close(self):
        if getattr(self, "_h", None):
            self._L.tsd_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != TSD_OK:
            _raise(rc, (self._L.tsd_group_last_error(self._h) or b"").decode())

    def set_series(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        self._check(self._L.tsd_group_series_set(self._h, x, len(x)))
        self.n = len(x)

    def counters(self, rank: int = 0) -> dict:
        c = Counters()
        self._check(self._L.tsd_get_counters(self._L.tsd_group_ctx(self._h, rank), C.byref(c)))
        return c.as_dict()

    def set_param(self, key: str, value: float):
        """Tuning knob on every rank (e.g. fused_peers=0: all-reduce kernels
        instead of fused peer stores)."""
        for r in range(self.size):
            rc = self._L.tsd_set_param(self._L.tsd_group_ctx(self._h, r), key.encode(), float(value))
            if rc != TSD_OK:
                _raise(rc, "set_param failed")

    def pardrag(self, m: int, r_sq: float, seglen: int) -> np.ndarray:
        N = max(self.n - m + 1, 1)
        out = np.zeros(N, RECORD_DTYPE)
        cnt = C.c_int64(0)
        self._check(self._L.tsd_group_pardrag(self._h, m, float(r_sq), seglen, out.ctypes.data, N, C.byref(cnt)))
        return out[: cnt.value].copy()

    def merlin_full(self, min_len: int, max_len: int, top_k: int = 1, seglen: int = 512,
                    max_retries: int = 100, reuse_stats: bool = True) -> MerlinReport:
        Ln = max(max_len - min_len + 1, 1)
        k = max(top_k, 1)
        counts = np.zeros(Ln, np.int64)
        recs = np.zeros((Ln, k), RECORD_DTYPE)
        final_r = np.zeros(Ln)
        retries = np.zeros(Ln, np.int64)
        failed = np.zeros(Ln, np.uint8)
        o = _Opts(top_k, seglen, 1, max_retries, 1 if reuse_stats else 0)
        self._check(self._L.tsd_group_merlin(self._h, min_len, max_len, C.byref(o), counts, recs.ctypes.data,
                                             final_r, retries, failed))
        rep = MerlinReport(min_len, max_len, final_r=final_r[:Ln], retries=retries[:Ln])
        for i in range(max_len - min_len + 1):
            if failed[i]:
                rep.failed_lengths.append(min_len + i)
            else:
                rep.per_length[min_len + i] = recs[i][: counts[i]].copy()
        return rep


_default: Engine | None = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(int(os.environ.get("TSD_DEVICE", "0")))
    return _default


def _with_series(x) -> Engine:
    e = default_engine()
    x = np.ascontiguousarray(x, dtype=np.float64)
    if e._series is None or len(e._series) != len(x) or not np.array_equal(e._series, x):
        e.set_series(x)
    return e


# reference-named module-level API -------------------------------------------
def init_stats(x, m: int):
    """stats.hpp:29 — (mu, sigma) for length m, computed on the GPU."""
    return _with_series(x).init_stats(m)


def advance_stats(x, m: int, mu, sigma):
    """stats.hpp:33 — Eq. 7-8 from length m to m+1 on the GPU."""
    return _with_series(x).advance_stats(m, mu, sigma)


def pardrag(x, m: int, r_sq: float, seglen: int, workers: int = 1, early_exit: bool = True):
    """pardrag.hpp:87-89 — range discords {i : nn(i)^2 >= r_sq}, sorted."""
    return _with_series(x).pardrag(m, r_sq, seglen)


def brute_force_nn(x, m: int):
    """drag.hpp:38 — exact nn^2 profile (GPU)."""
    return _with_series(x).brute_force_nn(m)


def merlin_full(x, min_len: int, max_len: int, top_k: int = 1, seglen: int = 512, workers: int = 1,
                max_retries: int = 100, reuse_stats: bool = True) -> MerlinReport:
    """merlin.hpp:50-51."""
    return _with_series(x).merlin_full(min_len, max_len, top_k, seglen, workers, max_retries,
                                       reuse_stats)


def merlin(x, min_len: int, max_len: int, top_k: int = 1, seglen: int = 512, workers: int = 1,
           max_retries: int = 100, reuse_stats: bool = True) -> MerlinReport:
    """merlin.hpp:53-54 (returns the report; .per_length / .failed_lengths)."""
    return merlin_full(x, min_len, max_len, top_k, seglen, workers, max_retries, reuse_stats)


def format_double(v: float) -> str:
    """io.cpp:42-46 shortest round-trip (Python repr is the same algorithm)."""
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") and "e" not in r else r


def discords_csv(per_length: dict) -> str:
    """write_discords_csv (io.cpp:121-130)."""
    lines = ["length,index,nn_dist,nn_dist_sq,score"]
    for m in sorted(per_length):
        for r in per_length[m]:
            lines.append(f"{m},{int(r['index'])},{format_double(r['nn_dist'])},"
                         f"{format_double(r['nn_dist_sq'])},{format_double(r['nn_dist_sq'] / (2.0 * m))}")
    return "\n".join(lines) + "\n"


def ranking_csv(ranking) -> str:
    """write_ranking_csv (heatmap.cpp:76-82)."""
    lines = ["rank,index,length,score"]
    for r, e in enumerate(ranking):
        lines.append(f"{r + 1},{int(e['index'])},{int(e['length'])},{format_double(e['score'])}")
    return "\n".join(lines) + "\n"


def read_discords_csv(text: str) -> dict:
    """read_discords_csv (io.cpp:132-160): {length: records} in file order."""
    out: dict = {}
    for no, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        if no == 1:
            if not line.startswith("length,"):
                raise RuntimeError(f"discord CSV: unexpected header '{line}'")
            continue
        f = line.split(",")
        if len(f) < 4:
            raise RuntimeError(f"discord CSV line {no}: expected at least 4 fields")
        try:
            m, idx, d, d2 = float(f[0]), float(f[1]), float(f[2]), float(f[3])
        except ValueError:
            raise RuntimeError(f"discord CSV line {no}: non-numeric field") from None
        out.setdefault(int(m), []).append((int(idx), d2, d))
    return {m: np.array(v, dtype=RECORD_DTYPE) for m, v in out.items()}
