"""Thin Python binding of libkvr.so (include/kvr.h): argument marshalling only.

Every step of the replay runs in the CUDA kernels behind the C ABI; this module
only converts Python values / torch tensors into the C structs and raw device
pointers.  PyTorch is used for device memory and streams.  There is no CPU
fallback: if libkvr.so is missing or no CUDA device is present the calls raise.

Function names mirror the C ABI (kvr_trace_load, kvr_sim_create, kvr_sim_run,
...).  ``DeviceTrace`` and ``Simulator`` are convenience owners of the torch
buffers those calls borrow.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVR_LIB", os.path.join(_PKG, "libkvr.so"))

EVICT_LRU, EVICT_RLT, EVICT_OPT = 0, 1, 2   # OPT: offline Belady, W = 1 (needs with_next_use)
RLT_EARLY_RESET, RLT_UNIFORM_LEAF, RLT_LRU_MARKED = 0, 1, 2
ROUTE_LBGR, ROUTE_STATIC_LINEAR, ROUTE_THRESHOLD, ROUTE_ROUND_ROBIN, ROUTE_RANDOM = 0, 1, 2, 3, 4
ROUTE_LBGR_RLS = 5   # LBGR, RLS reading of the 0.992 update (A8b)
ROUTE_CACHE_AWARE = 6   # SGLang-style cache-aware rule (A38)
MAX_TRACKER_LAG = 32
LEDGER_FIELDS = ("distinct", "misses", "first_misses", "clean")
TRIAL_OK, TRIAL_RING_OVERFLOW, TRIAL_VICTIM_LOG_FULL, TRIAL_BAD_POLICY = 0, 1, 2, 3
TRIAL_ADMISSION, TRIAL_BAD_TRACE = 4, 5
ERR_HASH_COLLISION = 4

# C-ABI entry points declared in include/kvr.h (the not-gpu test checks they are exported)
EXPORTS = ("kvr_last_error", "kvr_abi_version", "kvr_build_id", "kvr_trace_packed_bytes", "kvr_trace_load",
           "kvr_trace_info", "kvr_trace_chained_hashes", "kvr_trace_destroy",
           "kvr_trace_next_use_bytes", "kvr_trace_build_next_use", "kvr_trace_collision_bytes",
           "kvr_trace_check_collisions", "kvr_sim_create",
           "kvr_sim_destroy", "kvr_sim_plan", "kvr_sim_workspace_bytes",
           "kvr_sim_workspace_bytes_multi", "kvr_sim_run", "kvr_sim_run_multi",
           "kvr_trace_phase_bytes", "kvr_trace_build_phases", "kvr_sim_run_ledger")


class KvrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kvr status {status}: {msg}")
        self.status = status


class kvr_trace_desc(C.Structure):
    _fields_ = [("n_queries", C.c_uint32), ("block_tokens", C.c_uint32),
                ("hash_salt", C.c_uint64), ("n_blocks_total", C.c_uint64),
                ("arrival_ms", C.c_void_p), ("n_in_blocks", C.c_void_p),
                ("n_out_blocks", C.c_void_p), ("out_tokens", C.c_void_p),
                ("block_offsets", C.c_void_p), ("block_keys", C.c_void_p)]


class kvr_service_model(C.Structure):
    _fields_ = [("alpha_cached_ms", C.c_double), ("alpha_miss_ms", C.c_double),
                ("out_ms_per_token", C.c_double)]


class kvr_policy(C.Structure):
    _fields_ = [("eviction", C.c_uint32), ("rlt_fallback", C.c_uint32), ("router", C.c_uint32),
                ("_pad", C.c_uint32),
                ("est_alpha_cached_ms", C.c_double), ("est_alpha_miss_ms", C.c_double),
                ("rho", C.c_double), ("delta_t_ms", C.c_double), ("mu", C.c_double),
                ("theta0", C.c_double * 4), ("tau", C.c_double),
                ("w_hit", C.c_double), ("w_load", C.c_double), ("rls_p0", C.c_double),
                ("tracker_lag", C.c_uint32), ("tracker_grain", C.c_uint32),
                ("ca_balance_abs", C.c_double), ("ca_balance_rel", C.c_double),
                ("ca_cache_threshold", C.c_double), ("_pad2", C.c_uint64)]


class kvr_sim_config(C.Structure):
    _fields_ = [("W", C.c_uint32), ("capacity_blocks", C.c_uint32),
                ("truth", kvr_service_model), ("default_policy", kvr_policy),
                ("pending_ring", C.c_uint32), ("record_trials", C.c_uint32),
                ("latency_hist_bins", C.c_uint32), ("force_tier", C.c_uint32),
                ("extended_policies", C.c_uint32), ("batch_slots", C.c_uint32)]


POLICY_DTYPE = np.dtype([("eviction", "<u4"), ("rlt_fallback", "<u4"), ("router", "<u4"),
                         ("_pad", "<u4"), ("est_alpha_cached_ms", "<f8"),
                         ("est_alpha_miss_ms", "<f8"), ("rho", "<f8"), ("delta_t_ms", "<f8"),
                         ("mu", "<f8"), ("theta0", "<f8", (4,)), ("tau", "<f8"),
                         ("w_hit", "<f8"), ("w_load", "<f8"), ("rls_p0", "<f8"),
                         ("tracker_lag", "<u4"), ("tracker_grain", "<u4"),
                         ("ca_balance_abs", "<f8"), ("ca_balance_rel", "<f8"),
                         ("ca_cache_threshold", "<f8"), ("_pad2", "<u8")])
RESULT_DTYPE = np.dtype([(n, "<u8") for n in (
    "queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks", "evictions",
    "rlt_draws", "rlt_resets", "rlt_fallbacks", "max_pending", "decision_digest")] +
    [(n, "<f8") for n in ("sum_latency_ms", "sum_ttft_ms", "max_latency_ms", "makespan_ms",
                          "last_completion_ms", "sum_load_ms")] +
    [("status", "<i4"), ("_pad", "<u4")])
RECORD_DTYPE = np.dtype([("worker", "<u4"), ("hit_tokens", "<u4"), ("n_victims", "<u4"),
                         ("_pad", "<u4"), ("ttft_ms", "<f8"), ("latency_ms", "<f8"),
                         ("score", "<f8"), ("victim_offset", "<u8")])
assert POLICY_DTYPE.itemsize == C.sizeof(kvr_policy) == 160
assert RESULT_DTYPE.itemsize == 144 and RECORD_DTYPE.itemsize == 48

_lib = None


def lib():
    """Load libkvr.so; raise (no fallback) if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2601_18999_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, st = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
        L.kvr_last_error.restype = C.c_char_p
        L.kvr_abi_version.restype = u32
        L.kvr_build_id.restype = C.c_char_p
        sig = {
            "kvr_trace_packed_bytes": [vp, vp, vp],
            "kvr_trace_load": [vp, vp, C.c_size_t, vp, C.c_size_t, vp, vp],
            "kvr_trace_info": [vp, vp, vp, vp],
            "kvr_trace_chained_hashes": [vp, vp],
            "kvr_trace_destroy": [vp],
            "kvr_trace_next_use_bytes": [vp, vp, vp],
            "kvr_trace_collision_bytes": [vp, vp],
            "kvr_trace_check_collisions": [vp, vp, vp, C.c_size_t, vp, vp],
            "kvr_trace_build_next_use": [vp, vp, C.c_size_t, vp, C.c_size_t, vp, vp],
            "kvr_trace_phase_bytes": [vp, vp, vp],
            "kvr_trace_build_phases": [vp, u32, vp, C.c_size_t, vp, C.c_size_t, vp, vp, vp],
            "kvr_sim_run_ledger": [vp, vp, u32, vp, vp, vp, vp, vp, C.c_size_t, vp],
            "kvr_sim_create": [vp, vp],
            "kvr_sim_destroy": [vp],
            "kvr_sim_plan": [vp, u32, vp, vp, vp],
            "kvr_sim_workspace_bytes": [vp, vp, u32, vp],
            "kvr_sim_workspace_bytes_multi": [vp, u32, vp, u32, vp],
            "kvr_sim_run": [vp, vp, u32, vp, vp, vp, vp, vp, vp, u64, vp, C.c_size_t, vp],
            "kvr_sim_run_multi": [vp, u32, vp, vp, u32, vp, vp, vp, vp, vp, vp, u64, vp,
                                  C.c_size_t, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = st
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise KvrError(status, lib().kvr_last_error().decode(errors="replace"))


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return int(t.data_ptr())


def _stream_ptr(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream) or None


# ----------------------------------------------------------------- C-ABI mirrors
def kvr_abi_version() -> int:
    return int(lib().kvr_abi_version())


def kvr_last_error() -> str:
    return lib().kvr_last_error().decode(errors="replace")


def kvr_build_id() -> str:
    return lib().kvr_build_id().decode()


def kvr_trace_packed_bytes(desc: kvr_trace_desc):
    pb, sb = C.c_size_t(0), C.c_size_t(0)
    _check(lib().kvr_trace_packed_bytes(C.byref(desc), C.byref(pb), C.byref(sb)))
    return pb.value, sb.value


def kvr_trace_load(desc: kvr_trace_desc, packed, scratch, stream=None) -> int:
    h = C.c_void_p(0)
    _check(lib().kvr_trace_load(C.byref(desc), _ptr(packed), packed.numel() * packed.element_size(),
                                _ptr(scratch), scratch.numel() * scratch.element_size(),
                                _stream_ptr(stream), C.byref(h)))
    return h.value


def kvr_trace_info(handle: int):
    n, mx, tot = C.c_uint32(0), C.c_uint32(0), C.c_uint64(0)
    _check(lib().kvr_trace_info(handle, C.byref(n), C.byref(mx), C.byref(tot)))
    return n.value, mx.value, tot.value


def kvr_trace_chained_hashes(handle: int) -> int:
    p = C.c_void_p(0)
    _check(lib().kvr_trace_chained_hashes(handle, C.byref(p)))
    return p.value


def kvr_trace_destroy(handle: int):
    _check(lib().kvr_trace_destroy(handle))


def kvr_trace_next_use_bytes(handle: int):
    a, b = C.c_size_t(0), C.c_size_t(0)
    _check(lib().kvr_trace_next_use_bytes(handle, C.byref(a), C.byref(b)))
    return a.value, b.value


def kvr_trace_collision_bytes(handle: int) -> int:
    a = C.c_size_t(0)
    _check(lib().kvr_trace_collision_bytes(handle, C.byref(a)))
    return a.value


def kvr_trace_check_collisions(handle: int, block_keys, scratch, stream=None):
    """Returns (status, n_collisions); status KVR_ERR_HASH_COLLISION (4) is not raised."""
    n = C.c_uint64(0)
    st = lib().kvr_trace_check_collisions(handle, _ptr(block_keys), _ptr(scratch), scratch.numel(),
                                          _stream_ptr(stream), C.byref(n))
    if st not in (0, ERR_HASH_COLLISION):
        _check(st)
    return st, n.value


def kvr_trace_build_next_use(handle: int, nu, scratch, stream=None) -> int:
    h = C.c_void_p(0)
    _check(lib().kvr_trace_build_next_use(handle, _ptr(nu), nu.numel() * nu.element_size(),
                                          _ptr(scratch), scratch.numel(), _stream_ptr(stream),
                                          C.byref(h)))
    return h.value


def kvr_trace_phase_bytes(handle: int):
    a, b = C.c_size_t(0), C.c_size_t(0)
    _check(lib().kvr_trace_phase_bytes(handle, C.byref(a), C.byref(b)))
    return a.value, b.value


def kvr_trace_build_phases(handle: int, B: int, phase, scratch, stream=None):
    """Returns (new handle, n_phases)."""
    h = C.c_void_p(0)
    n = C.c_uint32(0)
    _check(lib().kvr_trace_build_phases(handle, B, _ptr(phase), phase.numel() * phase.element_size(),
                                        _ptr(scratch), scratch.numel(), _stream_ptr(stream),
                                        C.byref(n), C.byref(h)))
    return h.value, n.value


def kvr_sim_run_ledger(handle: int, trace: int, n_trials: int, keys, policies, results, ledger,
                       workspace, stream=None):
    _check(lib().kvr_sim_run_ledger(
        handle, trace, n_trials, _ptr(keys), _ptr(policies), _ptr(results), _ptr(ledger),
        _ptr(workspace), 0 if workspace is None else workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def kvr_sim_create(cfg: kvr_sim_config) -> int:
    h = C.c_void_p(0)
    _check(lib().kvr_sim_create(C.byref(cfg), C.byref(h)))
    return h.value


def kvr_sim_destroy(handle: int):
    _check(lib().kvr_sim_destroy(handle))


def kvr_sim_plan(handle: int, max_path_blocks: int):
    tier, smem, ctas = C.c_uint32(0), C.c_size_t(0), C.c_uint32(0)
    _check(lib().kvr_sim_plan(handle, max_path_blocks, C.byref(tier), C.byref(smem), C.byref(ctas)))
    return tier.value, smem.value, ctas.value


def kvr_sim_workspace_bytes_multi(handle: int, traces: Sequence[int], n_trials: int) -> int:
    arr = (C.c_void_p * len(traces))(*traces)
    b = C.c_size_t(0)
    _check(lib().kvr_sim_workspace_bytes_multi(handle, len(traces), arr, n_trials, C.byref(b)))
    return b.value


def kvr_sim_workspace_bytes(handle: int, trace: int, n_trials: int) -> int:
    b = C.c_size_t(0)
    _check(lib().kvr_sim_workspace_bytes(handle, trace, n_trials, C.byref(b)))
    return b.value


def kvr_sim_run_multi(handle: int, traces: Sequence[int], trial_trace, n_trials: int, keys,
                      policies, results, hist, records, victims, workspace, stream=None):
    arr = (C.c_void_p * len(traces))(*traces)
    _check(lib().kvr_sim_run_multi(
        handle, len(traces), arr, _ptr(trial_trace), n_trials, _ptr(keys), _ptr(policies),
        _ptr(results), _ptr(hist), _ptr(records), _ptr(victims),
        0 if victims is None else victims.numel(), _ptr(workspace),
        0 if workspace is None else workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


def kvr_sim_run(handle: int, trace: int, n_trials: int, keys, policies, results, hist, records,
                victims, workspace, stream=None):
    _check(lib().kvr_sim_run(
        handle, trace, n_trials, _ptr(keys), _ptr(policies), _ptr(results), _ptr(hist),
        _ptr(records), _ptr(victims), 0 if victims is None else victims.numel(), _ptr(workspace),
        0 if workspace is None else workspace.numel() * workspace.element_size(),
        _stream_ptr(stream)))


# ------------------------------------------------------------- buffer owners
@dataclass
class Policy:
    """Defaults = App. A under readings A8-A17."""
    eviction: int = EVICT_RLT
    rlt_fallback: int = RLT_EARLY_RESET
    router: int = ROUTE_LBGR
    est_alpha_cached_ms: float = 0.0
    est_alpha_miss_ms: float = 1.0
    rho: float = 31.0 / 32.0
    delta_t_ms: float = 20.0
    # NLMS step of router 0 (reading A8, revised r2: 1 - 0.992 = 0.008) or the RLS forgetting
    # factor of router 5 (A8b: 0.992); None = that router's default
    mu: Optional[float] = None
    theta0: Sequence[float] = (0.0, 0.0, 0.0, 0.0)
    tau: float = 1.5
    w_hit: float = 1.0
    w_load: float = 1.0
    rls_p0: float = 1000.0     # LBGR_RLS initial covariance P = rls_p0 * I
    tracker_lag: int = 0       # A29: router's h~ lags the last k queries' updates (k <= 32)
    tracker_grain: int = 1     # A29: router sees whole grains of matched blocks
    ca_balance_abs: float = 32.0        # A38 (ROUTE_CACHE_AWARE): imbalance iff max-min > abs
    ca_balance_rel: float = 1.0001      #   and max > rel * min (pending queries)
    ca_cache_threshold: float = 0.5     #   highest match if h~/|q| > threshold

    def mu_value(self) -> float:
        if self.mu is not None:
            return float(self.mu)
        return 0.992 if self.router == ROUTE_LBGR_RLS else 0.008

    def _get(self, f):
        return self.mu_value() if f == "mu" else getattr(self, f)

    def c(self) -> kvr_policy:
        p = kvr_policy()
        for f, _ in kvr_policy._fields_:
            if f in ("_pad", "_pad2"):
                continue
            if f == "theta0":
                for k in range(4):
                    p.theta0[k] = float(self.theta0[k])
            else:
                setattr(p, f, self._get(f))
        return p

    def row(self) -> np.ndarray:
        r = np.zeros((), dtype=POLICY_DTYPE)
        for f in POLICY_DTYPE.names:
            if f not in ("_pad", "_pad2"):
                r[f] = self._get(f)
        return r


def policies_extended(arr: np.ndarray) -> bool:
    """True if any policy needs the extended kernel (OPT, LBGR_RLS, CACHE_AWARE, tracker bias)."""
    a = np.asarray(arr).view(POLICY_DTYPE)
    return bool(np.any((a["eviction"] == EVICT_OPT) | (a["router"] == ROUTE_LBGR_RLS) |
                       (a["router"] == ROUTE_CACHE_AWARE) |
                       (a["tracker_lag"] != 0) | (a["tracker_grain"] != 1)))


def policies_array(pols: Sequence[Policy]) -> np.ndarray:
    a = np.zeros(len(pols), dtype=POLICY_DTYPE)
    for i, p in enumerate(pols):
        a[i] = p.row()
    return a


class DeviceTrace:
    """Raw trace uploaded to torch device tensors and packed by kvr_trace_load."""

    FIELDS = (("arrival", "arrival_ms", np.float64, np.float64),
              ("n_in", "n_in_blocks", np.uint32, np.int32),
              ("n_out", "n_out_blocks", np.uint32, np.int32),
              ("out_tokens", "out_tokens", np.uint32, np.int32),
              ("offsets", "block_offsets", np.uint64, np.int64),
              ("keys", "block_keys", np.uint64, np.int64))

    @staticmethod
    def pin(raw) -> dict:
        """Pinned host copies of the raw trace arrays (for timed host->device uploads).
        Unsigned arrays travel as same-width signed torch dtypes (bit patterns preserved)."""
        import torch
        out = {}
        for attr, name, src, dst in DeviceTrace.FIELDS:
            a = getattr(raw, name)
            if attr == "keys" and len(a) == 0:
                a = np.zeros(1, np.uint64)
            out[attr] = torch.from_numpy(np.ascontiguousarray(a.astype(src)).view(dst)).pin_memory()
        return out

    def __init__(self, raw, device="cuda", stream=None, host: Optional[dict] = None):
        import torch
        self.raw = raw
        self.device = torch.device(device)
        for attr, name, src, dst in self.FIELDS:
            if host is not None:
                t = host[attr]
            else:
                a = getattr(raw, name)
                if attr == "keys" and len(a) == 0:
                    a = np.zeros(1, np.uint64)
                t = torch.from_numpy(np.ascontiguousarray(a.astype(src)).view(dst))
            setattr(self, attr, t.to(device=self.device, non_blocking=True))
        d = kvr_trace_desc()
        d.n_queries = raw.n_queries
        d.block_tokens = raw.block_tokens
        d.hash_salt = raw.hash_salt
        d.n_blocks_total = raw.total_blocks
        d.arrival_ms = _ptr(self.arrival)
        d.n_in_blocks = _ptr(self.n_in)
        d.n_out_blocks = _ptr(self.n_out)
        d.out_tokens = _ptr(self.out_tokens)
        d.block_offsets = _ptr(self.offsets)
        d.block_keys = _ptr(self.keys)
        self.desc = d
        pb, sb = kvr_trace_packed_bytes(d)
        self.packed = torch.empty(pb, dtype=torch.uint8, device=self.device)
        self.scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        self.handle = kvr_trace_load(d, self.packed, self.scratch, stream)
        self.n_queries, self.max_path_blocks, self.n_blocks_total = kvr_trace_info(self.handle)

    def chained_hashes(self) -> np.ndarray:
        """Copy of the device identities H (for packer parity)."""
        import torch
        n = self.n_blocks_total
        off = kvr_trace_chained_hashes(self.handle) - _ptr(self.packed)
        return self.packed[off: off + 8 * n].cpu().numpy().view(np.uint64).copy()

    def identity_digest(self) -> int:
        """Order-sensitive checksum of the packed identities, computed on the device
        (multi-GPU check that every rank packed the same trace)."""
        import torch
        n = self.n_blocks_total
        if n == 0:
            return 0
        off = kvr_trace_chained_hashes(self.handle) - _ptr(self.packed)
        h = self.packed[off: off + 8 * n].view(torch.int64)
        pos = torch.arange(1, n + 1, dtype=torch.int64, device=h.device)
        return int((h.sum() + (h ^ (pos * 0x5851F42D4C957F2D)).sum()).item()) & 0xFFFFFFFFFFFFFFFF

    def collisions(self, stream=None) -> int:
        """Identity collision pairs of the loaded trace (kvr_trace_check_collisions); 0 = none."""
        import torch
        nb = kvr_trace_collision_bytes(self.handle)
        scratch = torch.empty(max(1, nb), dtype=torch.uint8, device=self.device)
        return kvr_trace_check_collisions(self.handle, self.keys, scratch, stream)[1]

    def with_next_use(self, stream=None) -> "DeviceTrace":
        """A trace handle that also carries the next-use index (offline OPT,
        KVR_EVICT_OPT): same packed buffer, plus a u32 [n_blocks_total] index
        built on the device by kvr_trace_build_next_use."""
        import copy
        import torch
        nb, sb = kvr_trace_next_use_bytes(self.handle)
        t = copy.copy(self)
        t.nu = torch.empty(max(1, nb // 4), dtype=torch.int32, device=self.device)
        scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=self.device)
        t.handle = kvr_trace_build_next_use(self.handle, t.nu, scratch, stream)
        torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()
        t._parent = self        # keeps the packed buffer alive
        return t

    def with_phases(self, B: int, stream=None) -> "DeviceTrace":
        """A trace handle that also carries the phase index of the phase ledger:
        phases of B distinct identities, first-appearance bits and next occurrences, built
        on the device by kvr_trace_build_phases (keeps this handle's next-use index)."""
        import copy
        import torch
        pb, sb = kvr_trace_phase_bytes(self.handle)
        t = copy.copy(self)
        t.phase = torch.empty(max(1, pb // 4), dtype=torch.int32, device=self.device)
        scratch = torch.empty(max(1, sb), dtype=torch.uint8, device=self.device)
        t.handle, t.n_phases = kvr_trace_build_phases(self.handle, B, t.phase, scratch, stream)
        t.phase_B = B
        t._parent = self
        return t

    def phase_index(self):
        """(ph, nx, distinct) copies: phase | first-appearance bit, next occurrence, per phase."""
        n = self.n_blocks_total
        a = self.phase.cpu().numpy().view(np.uint32)
        return a[:n].copy(), a[n:2 * n].copy(), a[2 * n: 2 * n + self.n_phases].copy()

    def next_use(self) -> np.ndarray:
        """Copy of the device next-use index (u32 per block occurrence, CSR order)."""
        return self.nu[: self.n_blocks_total].cpu().numpy().view(np.uint32).copy()

    def close(self):
        if getattr(self, "handle", None):
            kvr_trace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RunOutput:
    results: np.ndarray                 # RESULT_DTYPE [n_trials]
    records: Optional[np.ndarray]       # RECORD_DTYPE [record_trials, stride]
    victims: Optional[np.ndarray]       # u64 [victims_cap]
    hist: Optional[np.ndarray]          # u32 [n_trials, bins]


class Simulator:
    """kvr_sim handle plus its configuration (W, B, truth service model, policy)."""

    def __init__(self, W: int, capacity_blocks: int, policy: Optional[Policy] = None,
                 alpha_cached_ms: float = 0.0, alpha_miss_ms: float = 1.0,
                 out_ms_per_token: float = 20.0, pending_ring: int = 256,
                 record_trials: int = 0, latency_hist_bins: int = 0, force_tier: int = 0,
                 extended_policies: bool = False, batch_slots: int = 0):
        cfg = kvr_sim_config()
        cfg.W, cfg.capacity_blocks = W, capacity_blocks
        cfg.truth.alpha_cached_ms = alpha_cached_ms
        cfg.truth.alpha_miss_ms = alpha_miss_ms
        cfg.truth.out_ms_per_token = out_ms_per_token
        cfg.default_policy = (policy or Policy()).c()
        cfg.pending_ring, cfg.record_trials = pending_ring, record_trials
        cfg.latency_hist_bins, cfg.force_tier = latency_hist_bins, force_tier
        cfg.extended_policies = 1 if extended_policies else 0
        cfg.batch_slots = batch_slots   # 0: beta = 1 model; >= 1: continuous batching (A30-A36)
        self.cfg = cfg
        self.handle = kvr_sim_create(cfg)
        self._ws = None

    def _need_extended(self, policies: Optional[np.ndarray]):
        """Switch to the kernel instantiation with the extended policies when a
        per-trial policy array uses one (OPT, LBGR_RLS, tracker bias)."""
        if (policies is None or self.cfg.extended_policies or self.cfg.batch_slots
                or not policies_extended(policies)):
            return
        self.cfg.extended_policies = 1
        old = self.handle
        self.handle = kvr_sim_create(self.cfg)
        kvr_sim_destroy(old)

    def plan(self, max_path_blocks: int):
        return kvr_sim_plan(self.handle, max_path_blocks)

    def workspace(self, traces: Sequence[DeviceTrace], n_trials: int, device="cuda"):
        import torch
        nb = kvr_sim_workspace_bytes_multi(self.handle, [t.handle for t in traces], n_trials)
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=device)
        return self._ws

    def run(self, traces, keys, policies: Optional[np.ndarray] = None,
            trial_trace: Optional[np.ndarray] = None, victims_cap: int = 0, stream=None,
            sync: bool = True, buffers: Optional[dict] = None):
        """Launch kvr_sim_run(_multi); returns RunOutput (sync) or the device buffers."""
        import torch
        if isinstance(traces, DeviceTrace):
            traces = [traces]
        dev = traces[0].device
        n = len(keys)
        self._need_extended(policies)
        b = buffers if buffers is not None else self.alloc(traces, n, victims_cap, dev)
        if policies is not None:
            b["policies"].copy_(torch.from_numpy(np.ascontiguousarray(policies).view(np.uint8)))
        b["keys"].copy_(torch.from_numpy(np.asarray(keys, dtype=np.uint64).view(np.int64)))
        if trial_trace is not None:
            b["trial_trace"].copy_(torch.from_numpy(np.asarray(trial_trace, np.uint32).view(np.int32)))
        self.launch(traces, n, b, with_policies=policies is not None, stream=stream)
        if not sync:
            return b
        return self.collect(b, n)

    def alloc(self, traces, n, victims_cap=0, dev="cuda"):
        import torch
        R = min(self.cfg.record_trials, n)
        stride = max(t.n_queries for t in traces)
        bins = self.cfg.latency_hist_bins
        return {
            "keys": torch.empty(n, dtype=torch.int64, device=dev),
            "policies": torch.empty(n * POLICY_DTYPE.itemsize, dtype=torch.uint8, device=dev),
            "trial_trace": torch.zeros(n, dtype=torch.int32, device=dev),
            "results": torch.empty(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev),
            "records": torch.empty(max(1, R * stride) * RECORD_DTYPE.itemsize, dtype=torch.uint8,
                                   device=dev) if R else None,
            "victims": torch.zeros(victims_cap, dtype=torch.int64, device=dev)
            if (R and victims_cap) else None,
            "hist": torch.zeros(n * bins, dtype=torch.int32, device=dev) if bins else None,
            "workspace": self.workspace(traces, n, dev),
            "R": R, "stride": stride,
        }

    def launch(self, traces, n, b, with_policies=True, stream=None):
        kvr_sim_run_multi(self.handle, [t.handle for t in traces],
                          b["trial_trace"] if len(traces) > 1 else None, n, b["keys"],
                          b["policies"] if with_policies else None, b["results"], b["hist"],
                          b["records"], b["victims"], b["workspace"], stream)

    def collect(self, b, n) -> RunOutput:
        import torch
        torch.cuda.synchronize()
        res = b["results"].cpu().numpy().view(RESULT_DTYPE)[:n].copy()
        rec = None
        if b["records"] is not None:
            rec = b["records"].cpu().numpy().view(RECORD_DTYPE)[: b["R"] * b["stride"]]
            rec = rec.reshape(b["R"], b["stride"]).copy()
        vic = b["victims"].cpu().numpy().view(np.uint64).copy() if b["victims"] is not None else None
        hist = b["hist"].cpu().numpy().view(np.uint32).reshape(n, -1).copy() \
            if b["hist"] is not None else None
        return RunOutput(res, rec, vic, hist)

    def run_ledger(self, trace: DeviceTrace, keys, policies: Optional[np.ndarray] = None,
                   stream=None):
        """kvr_sim_run_ledger (W = 1, trace.with_phases(B)): returns (results, ledger)
        with ledger u32 [n_trials, n_phases, 4] = LEDGER_FIELDS per phase."""
        import torch
        dev = trace.device
        n = len(keys)
        if not self.cfg.extended_policies:
            self.cfg.extended_policies = 1
            old = self.handle
            self.handle = kvr_sim_create(self.cfg)
            kvr_sim_destroy(old)
        nph = getattr(trace, "n_phases", 0)   # 0: no phase index (the C ABI refuses it)
        npz = max(1, nph)
        kt = torch.from_numpy(np.asarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
        pt = (torch.from_numpy(np.ascontiguousarray(policies).view(np.uint8)).to(dev)
              if policies is not None else None)
        res = torch.empty(max(1, n) * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        led = torch.zeros(max(1, n * npz * 4), dtype=torch.int32, device=dev)
        ws = self.workspace([trace], n, dev)
        kvr_sim_run_ledger(self.handle, trace.handle, n, kt, pt, res, led, ws, stream)
        torch.cuda.synchronize()
        r = res.cpu().numpy().view(RESULT_DTYPE)[:n].copy()
        lg = led.cpu().numpy().view(np.uint32)[: n * nph * 4]
        return r, lg.reshape(n, nph, 4).copy()

    def close(self):
        if getattr(self, "handle", None):
            kvr_sim_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
