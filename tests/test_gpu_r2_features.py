"""GPU parity of the round-2 SURVEY §8(f) rows against the oracle (pins P38-P40):

* KVR_ROUTE_CACHE_AWARE, the SGLang-style cache-aware rule (reading A38), in
  both engines, every branch exercised (imbalanced / highest match / fewest blocks);
* the k-event stale tracker (App. E, reading A29, k = 1..32) through the mirror of
  each worker's cache, both state tiers, with every router;
* the phase ledger (reading A39): the device phase partition against the
  oracle's and an independent Python split, and per-phase misses / first-appearance
  misses / clean tokens of L-LRU, RLT and OPT trials equal to the oracle's ledger.
"""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import compare, compare_batched

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvr():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr as k
    k.lib()
    return k


# ------------------------------------------------------------------ cache-aware (A38)
CA_SETTINGS = [dict(), dict(ca_balance_abs=1.0, ca_balance_rel=1.2),
               dict(ca_balance_abs=4.0, ca_balance_rel=1.0001, ca_cache_threshold=0.2),
               dict(ca_balance_abs=1e18, ca_cache_threshold=0.9),
               dict(ca_balance_abs=-1.0, ca_balance_rel=0.0)]


@pytest.mark.parametrize("W", [2, 4, 8, 16, 32])
def test_cache_aware_parity(kvr, oracle_mod, W):
    tr = wl.gsp(20, 12, 0.5, seed=0xA0 + W, W=W, util=2.0, lengths=(128, 256, 512))
    pols = [kvr.Policy(router=kvr.ROUTE_CACHE_AWARE, eviction=k % 2, **kw)
            for k, kw in enumerate(CA_SETTINGS)]
    out, _ = compare(oracle_mod, kvr, tr, W, 512, pols, list(range(1, len(pols) + 1)),
                     ring=tr.n_queries)
    # every branch was taken somewhere: imbalance routing differs from the affinity one
    workers = [tuple(out.records[t]["worker"][: tr.n_queries]) for t in range(len(pols))]
    assert len(set(workers)) >= 3


@pytest.mark.parametrize("tier", [1, 2])
def test_cache_aware_tiers_drift(kvr, oracle_mod, tier):
    tr = wl.drift(2048, 200_000, seed=0xC5, W=16).prefix(2500)
    pols = [kvr.Policy(router=kvr.ROUTE_CACHE_AWARE, eviction=e, **kw)
            for e in (0, 1) for kw in (dict(), dict(ca_balance_abs=2.0, ca_cache_threshold=0.3))]
    compare(oracle_mod, kvr, tr, 16, 512, pols, [5, 6, 7, 8], force_tier=tier, ring=tr.n_queries)


@pytest.mark.parametrize("beta", [1, 2, 4])
def test_cache_aware_batching(kvr, oracle_mod, beta):
    tr = wl.gsp(16, 10, 0.5, seed=0xA7 + beta, W=4, util=2.0, lengths=(128, 256))
    pols = [kvr.Policy(router=kvr.ROUTE_CACHE_AWARE, eviction=k % 2, **kw)
            for k, kw in enumerate(CA_SETTINGS)]
    compare_batched(oracle_mod, kvr, tr, 4, 256, beta, pols, list(range(1, len(pols) + 1)),
                    ring=tr.n_queries)


def test_cache_aware_closed_form_jsq(kvr, oracle_mod):
    """P38 through the GPU: abs = -1, rel = 0, arrivals at 0 -> join-shortest-queue."""
    paths = [[100 * j + d for d in range(4)] for j in range(12)]
    tr = wl.from_paths(paths, arrival_ms=[0.0] * 12)
    out, _ = compare(oracle_mod, kvr, tr, 3, 64,
                     [kvr.Policy(router=kvr.ROUTE_CACHE_AWARE, ca_balance_abs=-1.0,
                                 ca_balance_rel=0.0, eviction=0)], [1])
    assert list(out.records[0]["worker"][:12]) == [j % 3 for j in range(12)]


# ------------------------------------------------------------ k-event stale tracker (A29)
@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("tier", [1, 2])
def test_tracker_lag_k_parity(kvr, oracle_mod, W, tier):
    tr = wl.gsp(20, 10, 0.5, seed=0xB0 + W, W=W, lengths=(128, 256, 512))
    pols = []
    for r, lag in ((0, 2), (1, 3), (2, 5), (6, 4), (0, 32), (1, 1), (2, 17)):
        pols.append(kvr.Policy(router=r, tracker_lag=lag, eviction=lag % 2,
                               tracker_grain=1 if lag != 5 else 4, w_hit=1.0, w_load=0.5))
    compare(oracle_mod, kvr, tr, W, 512, pols, list(range(40, 40 + len(pols))), force_tier=tier,
            ring=tr.n_queries)


@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_tracker_lag_closed_form(kvr, oracle_mod, k):
    """P39 through the GPU: anti-affinity on one repeated path gives
    [0]*(k+1) + [1]*(k+1) + [0]*... exactly."""
    n = 4 * k + 6
    tr = wl.from_paths([[5, 6, 7, 8]] * n, arrival_ms=[1e6 * j for j in range(n)])
    pol = kvr.Policy(router=1, w_load=0.0, w_hit=-1.0, tracker_lag=k, eviction=0)
    out, _ = compare(oracle_mod, kvr, tr, 2, 64, [pol], [1])
    assert list(out.records[0]["worker"][:n]) == [0] * (k + 1) + [1] * (k + 1) + [0] * (n - 2 * k - 2)


def test_tracker_lag_long_trace_rebuilds(kvr, oracle_mod):
    """A long trace at a small cache: the mirrors' tables fill with tombstones and are
    rebuilt many times; the lagged routing still equals the oracle's."""
    tr = wl.gsp(40, 40, 0.3, seed=0xB9, W=4, lengths=(128, 256))
    pols = [kvr.Policy(router=r, tracker_lag=lag, eviction=e)
            for r, lag, e in ((0, 8, 1), (2, 3, 0), (6, 12, 1))]
    compare(oracle_mod, kvr, tr, 4, 96, pols, [3, 4, 5], ring=tr.n_queries)


# ----------------------------------------------------------------- phase ledger (A39)
def _ledger_case(kvr, oracle_mod, tr, B, evictions, keys):
    from oracle import analysis as an
    dt = kvr.DeviceTrace(tr)
    if kvr.EVICT_OPT in evictions:
        dt = dt.with_next_use()
    dtp = dt.with_phases(B)
    ph, nx, distinct = dtp.phase_index()
    ids = an.flattened_ids(tr)
    parts = an.phases(ids, B)
    assert dtp.n_phases == len(parts)
    starts = np.array([a for a, _ in parts])
    phase_of = np.searchsorted(starts, np.arange(len(ids)), side="right") - 1
    assert np.array_equal(ph & 0x7FFFFFFF, phase_of.astype(np.uint32))
    assert [int(x) for x in distinct] == [len(set(ids[a:b].tolist())) for a, b in parts]
    sim = kvr.Simulator(1, B, extended_policies=True, pending_ring=tr.n_queries)
    pols = kvr.policies_array([kvr.Policy(eviction=e, router=3) for e in evictions])
    res, led = sim.run_ledger(dtp, np.asarray(keys, np.uint64), pols)
    assert np.all(res["status"] == 0)
    for t, (e, k) in enumerate(zip(evictions, keys)):
        o = oracle_mod.phase_ledger(tr, B, e, philox_key=int(k))
        assert led[t].shape == o.shape
        if not np.array_equal(led[t], o):
            v = int(np.nonzero(np.any(led[t] != o, axis=1))[0][0])
            raise AssertionError(f"eviction {e} key {k}: phase {v} gpu {led[t][v]} oracle {o[v]}")
    return led


@pytest.mark.parametrize("B", [64, 1024])
def test_phase_ledger_adv(kvr, oracle_mod, B):
    """Config 4's Thm 1 family: L-LRU B-L+1 misses and 1 clean tail per steady phase,
    OPT one miss, RLT the marking bound; GPU ledger == oracle ledger."""
    tr = wl.adv(B, 4, 6, seed=0xC6)
    led = _ledger_case(kvr, oracle_mod, tr, B, [0, 1, 1, 2], [1, 2, 3, 4])
    assert np.all(led[0][1:-1, 1] == B - 3) and np.all(led[0][1:-1, 3] == 1)
    assert np.all(led[3][1:-1, 1] == 1)


@pytest.mark.parametrize("seed", range(4))
def test_phase_ledger_random_trees(kvr, oracle_mod, seed):
    tr = wl.random_tree(400, seed=0xD0 + seed, max_len=7, alphabet=3)
    _ledger_case(kvr, oracle_mod, tr, 12, [0, 1, 1, 1, 2], [5, 6, 7, 8, 9])


def test_phase_ledger_gsp_both_tiers(kvr, oracle_mod):
    """GSP-shaped paths (hundreds of blocks) at B = 512 (shared-memory tier) and B = 2048
    (global tier)."""
    tr = wl.gsp(12, 10, 0.5, seed=0xD7, W=1, lengths=(128, 256, 512))
    for B in (512, 2048):
        _ledger_case(kvr, oracle_mod, tr, B, [0, 1, 2], [11, 12, 13])


def test_phase_ledger_validation(kvr):
    tr = wl.adv(64, 4, 2, seed=1)
    dt = kvr.DeviceTrace(tr)
    sim = kvr.Simulator(1, 64, extended_policies=True)
    with pytest.raises(kvr.KvrError):           # no phase index
        sim.run_ledger(dt, np.array([1], np.uint64))
    with pytest.raises(kvr.KvrError):           # phases built for another B
        sim.run_ledger(dt.with_phases(32), np.array([1], np.uint64))
    with pytest.raises(kvr.KvrError):           # W must be 1
        kvr.Simulator(2, 64, extended_policies=True).run_ledger(dt.with_phases(64), np.array([1], np.uint64))


# -------------------------------------------------- split tier, two workers per warp
@pytest.mark.parametrize("W", [17, 24, 31, 32])
def test_split_tier_two_workers_per_warp(kvr, oracle_mod, W):
    """W > 16 runs ceil(W/2) warps of two workers (odd W leaves one warp with a single
    worker), in the shared-memory tier when it fits (W = 17 here) and otherwise the split
    tier (identities + tables in global memory, tree arrays / bitmaps / stamps in shared
    memory).  Every field, record and victim equals the oracle's, lean and extended
    policies, for the automatic tier, the forced split tier and the all-global tier 2."""
    tr = wl.gsp(24, 10, 0.5, seed=0xE0 + W, W=W, util=1.5, lengths=(128, 256, 512))
    sim = kvr.Simulator(W, 512)
    assert sim.plan(tr.max_blocks)[0] == (1 if W == 17 else 3)
    pols = [kvr.Policy(eviction=e, router=r) for e in (0, 1) for r in (0, 1, 2)]
    keys = list(range(60, 60 + len(pols)))
    for tier in (0, 2, 3):
        compare(oracle_mod, kvr, tr, W, 512, pols, keys, force_tier=tier, ring=tr.n_queries)
    ext = [kvr.Policy(eviction=1, router=6), kvr.Policy(eviction=0, tracker_lag=3),
           kvr.Policy(eviction=1, router=5), kvr.Policy(eviction=1, rlt_fallback=2)]
    compare(oracle_mod, kvr, tr, W, 512, ext, [70, 71, 72, 73], ring=tr.n_queries)


def test_split_tier_full_wave_every_trial(kvr, oracle_mod):
    """The two-workers-per-warp tier under a full resident wave and more: 200 trials (> 148
    CTAs) of W = 32 at B = 512 on one prefix-sharing trace, RLT and L-LRU mixed, every
    trial's result bytes equal to the oracle's.  Guards the cross-warp apply / score
    ordering (a worker updated by a non-home warp is scored by its home warp only after
    that apply finished): the race it replaced showed up only under concurrent trials."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array
    from parity_util import assert_result_equal, to_oracle_policy
    W, B, n = 32, 512, 200
    tr = wl.gsp(40, 40, 0.7, seed=0x5E1, W=W, util=0.8, lengths=(256, 512, 1024))
    pols = [Policy(eviction=t % 2) for t in range(n)]
    keys = np.arange(1, n + 1, dtype=np.uint64)
    sim = Simulator(W, B, pending_ring=4096)
    assert sim.plan(tr.max_blocks)[0] == 3   # the split tier
    out = sim.run(DeviceTrace(tr), keys, policies_array(pols))
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=B, pending_ring=4096)

    def one(t):
        return oracle_mod.run(cfg, tr, to_oracle_policy(oracle_mod, pols[t]), int(keys[t]))

    with ThreadPoolExecutor(max_workers=16) as ex:
        orc = list(ex.map(one, range(n)))
    for t, o in enumerate(orc):
        assert o.rc == 0
        assert_result_equal(out.results[t], o.result, f"W=32 split trial {t}")
