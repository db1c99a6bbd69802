"""CPU oracle for the replay of arxiv 2601.18999's online process.

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2601_18999_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``kvr_oracle.cpp`` (plain C++17, single threaded,
``-O2 -ffp-contract=off -fno-fast-math``); this module is the ctypes binding.
Functions without an independent pin are listed under "parity unpinned" in
DESIGN.md.
"""
from .binding import (  # noqa: F401
    EVICT_LRU, EVICT_RLT, EVICT_OPT,
    RLT_EARLY_RESET, RLT_UNIFORM_LEAF, RLT_LRU_MARKED,
    ROUTE_LBGR, ROUTE_STATIC_LINEAR, ROUTE_THRESHOLD, ROUTE_ROUND_ROBIN, ROUTE_RANDOM,
    ROUTE_LBGR_RLS, ROUTE_CACHE_AWARE, MAX_TRACKER_LAG, LEDGER_FIELDS,
    OracleConfig, OraclePolicy, build_oracle, lib,
    fmix64, philox4x32_10, chain, run, single_replay, bruteforce_min_misses, rls_step,
    rlt_exact_expectation, count_collisions, phase_ledger,
)
