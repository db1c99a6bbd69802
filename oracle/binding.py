"""ctypes binding of oracle/libkvr_oracle.so (TEST INFRASTRUCTURE, see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libkvr_oracle.so")
_SRC = os.path.join(_HERE, "kvr_oracle.cpp")
_HDR = os.path.join(_HERE, "kvr_oracle.h")

EVICT_LRU, EVICT_RLT, EVICT_OPT = 0, 1, 2
RLT_EARLY_RESET, RLT_UNIFORM_LEAF, RLT_LRU_MARKED = 0, 1, 2
ROUTE_LBGR, ROUTE_STATIC_LINEAR, ROUTE_THRESHOLD, ROUTE_ROUND_ROBIN, ROUTE_RANDOM = 0, 1, 2, 3, 4
ROUTE_LBGR_RLS = 5   # LBGR with the RLS reading of the 0.992 update (A8b)
ROUTE_CACHE_AWARE = 6   # SGLang-style cache-aware rule (A38)
MAX_TRACKER_LAG = 32


def build_oracle(force: bool = False) -> str:
    """Compile the oracle (plain g++, no CUDA).  Building the checker is not using it."""
    stale = (not os.path.exists(_SO) or
             os.path.getmtime(_SO) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", "-o", _SO + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Trace(C.Structure):
    _fields_ = [("n_queries", C.c_uint32), ("block_tokens", C.c_uint32),
                ("hash_salt", C.c_uint64),
                ("arrival_ms", C.c_void_p), ("n_in_blocks", C.c_void_p),
                ("n_out_blocks", C.c_void_p), ("out_tokens", C.c_void_p),
                ("block_offsets", C.c_void_p), ("block_keys", C.c_void_p)]


class _Policy(C.Structure):
    _fields_ = [("eviction", C.c_uint32), ("rlt_fallback", C.c_uint32), ("router", C.c_uint32),
                ("_pad", C.c_uint32),
                ("est_alpha_cached_ms", C.c_double), ("est_alpha_miss_ms", C.c_double),
                ("rho", C.c_double), ("delta_t_ms", C.c_double), ("mu", C.c_double),
                ("theta0", C.c_double * 4), ("tau", C.c_double),
                ("w_hit", C.c_double), ("w_load", C.c_double), ("rls_p0", C.c_double),
                ("tracker_lag", C.c_uint32), ("tracker_grain", C.c_uint32),
                ("ca_balance_abs", C.c_double), ("ca_balance_rel", C.c_double),
                ("ca_cache_threshold", C.c_double), ("_pad2", C.c_uint64)]


class _Config(C.Structure):
    _fields_ = [("W", C.c_uint32), ("capacity_blocks", C.c_uint32),
                ("alpha_cached_ms", C.c_double), ("alpha_miss_ms", C.c_double),
                ("out_ms_per_token", C.c_double),
                ("pending_ring", C.c_uint32), ("latency_hist_bins", C.c_uint32),
                ("batch_slots", C.c_uint32), ("_pad", C.c_uint32)]


class _Result(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks", "evictions",
        "rlt_draws", "rlt_resets", "rlt_fallbacks", "max_pending", "decision_digest")] + \
        [(n, C.c_double) for n in (
            "sum_latency_ms", "sum_ttft_ms", "max_latency_ms", "makespan_ms",
            "last_completion_ms", "sum_load_ms")] + [("status", C.c_int32), ("_pad", C.c_uint32)]


RECORD_DTYPE = np.dtype([("worker", "<u4"), ("hit_tokens", "<u4"), ("n_victims", "<u4"),
                         ("_pad", "<u4"), ("ttft_ms", "<f8"), ("latency_ms", "<f8"),
                         ("score", "<f8"), ("victim_offset", "<u8")])

_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_SO)
        L.kvro_fmix64.restype = C.c_uint64
        L.kvro_fmix64.argtypes = [C.c_uint64]
        L.kvro_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.kvro_chain.argtypes = [C.POINTER(_Trace), C.c_void_p]
        L.kvro_count_collisions.argtypes = [C.POINTER(_Trace), C.POINTER(C.c_uint64)]
        L.kvro_rls_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double]
        L.kvro_rls_step.restype = None
        L.kvro_run.argtypes = [C.POINTER(_Config), C.POINTER(_Trace), C.POINTER(_Policy),
                               C.c_uint64, C.POINTER(_Result), C.c_void_p, C.c_void_p,
                               C.c_uint64, C.c_void_p, C.c_int]
        L.kvro_single_replay.argtypes = [C.POINTER(_Trace), C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, C.c_void_p, C.POINTER(C.c_uint64),
                                         C.c_void_p, C.c_void_p, C.c_uint32,
                                         C.POINTER(C.c_uint32)]
        L.kvro_phase_ledger.argtypes = [C.POINTER(_Trace), C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_uint64, C.c_void_p, C.c_uint32,
                                        C.POINTER(C.c_uint32)]
        L.kvro_bruteforce_min_misses.argtypes = [C.POINTER(_Trace), C.c_uint32,
                                                 C.POINTER(C.c_uint64)]
        L.kvro_rlt_exact_expectation.argtypes = [C.POINTER(_Trace), C.c_uint32, C.c_uint32,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_uint64)]
        _lib = L
    return _lib


@dataclass
class OraclePolicy:
    """One replay's policy.  Defaults = App. A with the readings A8-A17."""
    eviction: int = EVICT_RLT
    rlt_fallback: int = RLT_EARLY_RESET
    router: int = ROUTE_LBGR
    est_alpha_cached_ms: float = 0.0
    est_alpha_miss_ms: float = 1.0
    rho: float = 31.0 / 32.0
    delta_t_ms: float = 20.0
    # NLMS step of router 0 (A8, revised r2: 1 - 0.992 = 0.008) or the RLS forgetting
    # factor of router 5 (A8b: 0.992); None = that router's default
    mu: Optional[float] = None
    theta0: Sequence[float] = (0.0, 0.0, 0.0, 0.0)
    tau: float = 1.5
    w_hit: float = 1.0
    w_load: float = 1.0
    rls_p0: float = 1000.0
    tracker_lag: int = 0       # A29: router lags the last k queries' updates
    tracker_grain: int = 1     # A29: router sees whole grains of matched blocks
    ca_balance_abs: float = 32.0        # A38 (router 6): imbalance iff max-min > abs
    ca_balance_rel: float = 1.0001      #   and max > rel * min (pending queries)
    ca_cache_threshold: float = 0.5     #   highest match if h~/|q| > threshold

    def _c(self) -> _Policy:
        p = _Policy()
        p.eviction, p.rlt_fallback, p.router = self.eviction, self.rlt_fallback, self.router
        p.est_alpha_cached_ms, p.est_alpha_miss_ms = self.est_alpha_cached_ms, self.est_alpha_miss_ms
        mu = self.mu if self.mu is not None else (0.992 if self.router == ROUTE_LBGR_RLS else 0.008)
        p.rho, p.delta_t_ms, p.mu = self.rho, self.delta_t_ms, float(mu)
        for k in range(4):
            p.theta0[k] = float(self.theta0[k])
        p.tau, p.w_hit, p.w_load = self.tau, self.w_hit, self.w_load
        p.rls_p0 = self.rls_p0
        p.tracker_lag, p.tracker_grain = self.tracker_lag, self.tracker_grain
        p.ca_balance_abs, p.ca_balance_rel = self.ca_balance_abs, self.ca_balance_rel
        p.ca_cache_threshold = self.ca_cache_threshold
        return p


@dataclass
class OracleConfig:
    W: int = 4
    capacity_blocks: int = 512
    alpha_cached_ms: float = 0.0
    alpha_miss_ms: float = 1.0
    out_ms_per_token: float = 20.0
    pending_ring: int = 256
    latency_hist_bins: int = 0
    batch_slots: int = 0       # 0: beta = 1 model (A3/A12); >= 1: continuous batching (A30-A35)

    def _c(self) -> _Config:
        c = _Config()
        c.W, c.capacity_blocks = self.W, self.capacity_blocks
        c.alpha_cached_ms, c.alpha_miss_ms = self.alpha_cached_ms, self.alpha_miss_ms
        c.out_ms_per_token = self.out_ms_per_token
        c.pending_ring, c.latency_hist_bins = self.pending_ring, self.latency_hist_bins
        c.batch_slots = self.batch_slots
        return c


class _TraceArgs:
    """Keeps the contiguous numpy arrays alive while the C struct points at them."""

    def __init__(self, tr):
        self.arrival = np.ascontiguousarray(tr.arrival_ms, dtype=np.float64)
        self.n_in = np.ascontiguousarray(tr.n_in_blocks, dtype=np.uint32)
        self.n_out = np.ascontiguousarray(tr.n_out_blocks, dtype=np.uint32)
        self.out_tokens = np.ascontiguousarray(tr.out_tokens, dtype=np.uint32)
        self.offsets = np.ascontiguousarray(tr.block_offsets, dtype=np.uint64)
        self.keys = np.ascontiguousarray(tr.block_keys, dtype=np.uint64)
        t = _Trace()
        t.n_queries = len(self.n_in)
        t.block_tokens = int(tr.block_tokens)
        t.hash_salt = int(tr.hash_salt)
        t.arrival_ms = self.arrival.ctypes.data
        t.n_in_blocks = self.n_in.ctypes.data
        t.n_out_blocks = self.n_out.ctypes.data
        t.out_tokens = self.out_tokens.ctypes.data
        t.block_offsets = self.offsets.ctypes.data
        t.block_keys = self.keys.ctypes.data if len(self.keys) else None
        self.c = t


def fmix64(x: int) -> int:
    return int(lib().kvro_fmix64(C.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def philox4x32_10(ctr: Sequence[int], key: Sequence[int]) -> tuple:
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().kvro_philox4x32_10(c.ctypes.data, k.ctypes.data, o.ctypes.data)
    return tuple(int(v) for v in o)


def count_collisions(tr) -> int:
    a = _TraceArgs(tr)
    out = C.c_uint64(0)
    rc = lib().kvro_count_collisions(C.byref(a.c), C.byref(out))
    if rc:
        raise ValueError(f"kvro_count_collisions rc={rc}")
    return int(out.value)


def rls_step(P: np.ndarray, theta: np.ndarray, phi, e: float, lam: float):
    """In-place RLS step (P float64 [4,4] C-contiguous, theta float64 [4])."""
    ph = np.ascontiguousarray(phi, dtype=np.float64)
    lib().kvro_rls_step(P.ctypes.data, theta.ctypes.data, ph.ctypes.data, float(e), float(lam))


def chain(tr) -> np.ndarray:
    a = _TraceArgs(tr)
    out = np.zeros(max(1, int(a.offsets[-1])), dtype=np.uint64)
    rc = lib().kvro_chain(C.byref(a.c), out.ctypes.data)
    if rc:
        raise ValueError(f"kvro_chain failed rc={rc}")
    return out[: int(a.offsets[-1])]


@dataclass
class OracleRun:
    result: dict
    records: Optional[np.ndarray] = None
    victims: Optional[np.ndarray] = None
    hist: Optional[np.ndarray] = None
    rc: int = 0


def run(cfg: OracleConfig, tr, pol: OraclePolicy, philox_key: int, record: bool = False,
        victims_cap: int = 0, check_invariants: bool = False) -> OracleRun:
    a = _TraceArgs(tr)
    res = _Result()
    n = len(a.n_in)
    recs = np.zeros(n, dtype=RECORD_DTYPE) if record else None
    vic = np.zeros(max(1, victims_cap), dtype=np.uint64) if (record and victims_cap) else None
    hist = np.zeros(cfg.latency_hist_bins, dtype=np.uint32) if cfg.latency_hist_bins else None
    c = cfg._c()
    p = pol._c()
    rc = lib().kvro_run(C.byref(c), C.byref(a.c), C.byref(p), C.c_uint64(philox_key),
                        C.byref(res),
                        recs.ctypes.data if recs is not None else None,
                        vic.ctypes.data if vic is not None else None,
                        C.c_uint64(victims_cap if vic is not None else 0),
                        hist.ctypes.data if hist is not None else None,
                        1 if check_invariants else 0)
    d = {f[0]: getattr(res, f[0]) for f in _Result._fields_ if not f[0].startswith("_")}
    return OracleRun(d, recs, vic, hist, rc)


def single_replay(tr, B: int, eviction: int, fallback: int = RLT_EARLY_RESET,
                  philox_key: int = 0):
    """Returns (total_misses, miss_flags[u8 per flattened block access])."""
    a = _TraceArgs(tr)
    total = int(a.offsets[-1])
    flags = np.zeros(max(1, total), dtype=np.uint8)
    tm = C.c_uint64(0)
    nd = C.c_uint32(0)
    rc = lib().kvro_single_replay(C.byref(a.c), B, eviction, fallback, C.c_uint64(philox_key),
                                  flags.ctypes.data, C.byref(tm), None, None, 0, C.byref(nd))
    if rc:
        raise ValueError(f"kvro_single_replay rc={rc}")
    return int(tm.value), flags[:total]


LEDGER_FIELDS = ("distinct", "misses", "first_misses", "clean")


def phase_ledger(tr, B: int, eviction: int, fallback: int = RLT_EARLY_RESET,
                 philox_key: int = 0) -> np.ndarray:
    """Per-phase ledger of one single-cache replay (A39): u32 array
    [n_phases, 4] of (distinct, misses, first_misses, clean); old-token misses are
    misses - first_misses."""
    a = _TraceArgs(tr)
    n = C.c_uint32(0)
    rc = lib().kvro_phase_ledger(C.byref(a.c), B, eviction, fallback, C.c_uint64(philox_key),
                                 None, 0, C.byref(n))
    if rc not in (0, 1, 3):
        raise ValueError(f"kvro_phase_ledger rc={rc}")
    out = np.zeros((max(1, n.value), 4), dtype=np.uint32)
    rc = lib().kvro_phase_ledger(C.byref(a.c), B, eviction, fallback, C.c_uint64(philox_key),
                                 out.ctypes.data, n.value, C.byref(n))
    if rc:
        raise ValueError(f"kvro_phase_ledger rc={rc}")
    return out[: n.value]


def bruteforce_min_misses(tr, B: int) -> int:
    a = _TraceArgs(tr)
    out = C.c_uint64(0)
    rc = lib().kvro_bruteforce_min_misses(C.byref(a.c), B, C.byref(out))
    if rc:
        raise ValueError(f"kvro_bruteforce_min_misses rc={rc}")
    return int(out.value)


def rlt_exact_expectation(tr, B: int, fallback: int = RLT_EARLY_RESET):
    """Exact (mean, variance, leaves) of RLT misses over every uniform choice."""
    a = _TraceArgs(tr)
    m1, m2, nl = C.c_double(0), C.c_double(0), C.c_uint64(0)
    rc = lib().kvro_rlt_exact_expectation(C.byref(a.c), B, fallback, C.byref(m1), C.byref(m2),
                                          C.byref(nl))
    if rc:
        raise ValueError(f"kvro_rlt_exact_expectation rc={rc}")
    return m1.value, m2.value - m1.value * m1.value, int(nl.value)
