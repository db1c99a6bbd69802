"""GPU parity at BASELINE.json sizes (SURVEY §8(d) recipes), field by field against the
oracle's full replay of the same trial.

* config 2: the exact launch `bench.py --workload c2` times (3 x 100k-query GSP traces,
  W = 8, B = 512, 1,024 trials in one kvr_sim_run_multi); one trial of each of the six
  (trace, eviction) classes replayed by the oracle over all 100k queries.
* config 3: DRIFT(8192, 1M, 1.1), W = 16, RLT: a 100k-query prefix for each router
  (LBGR at App. A, STATIC, THRESHOLD) plus the collapsing NLMS cell (mu = 0.992, dt = 10
  ms) whose queues grow to tens of thousands of pending completions; every record and
  every victim compared.
* config 4: Thm 1 adversarial family, W = 1, B in {64, 1024, 4096}, full length.
* config 5: one trial of EVERY one of the 48 cells at recipe size (GSP(128,32,r),
  MT(128,r) x2, LD(512,Q_d) incl. LD-high with 16,384 queries; W in {4, 8, 16, 32}),
  launched exactly as bench.py does (one launch per W over the 12 traces), with the
  trial keys of the fixed 65,536 list; records and victims compared.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import assert_records_equal, assert_result_equal, compare, to_oracle_policy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvr():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr as k
    return k


def _oracle_many(oracle_mod, jobs):
    """jobs: [(cfg, trace, OraclePolicy, key, record, victims_cap)] on host threads."""
    def one(j):
        cfg, tr, pol, key, record, vcap = j
        r = oracle_mod.run(cfg, tr, pol, key, record=record, victims_cap=vcap)
        assert r.rc == 0, r.rc
        return r
    with ThreadPoolExecutor(max_workers=16) as ex:
        return list(ex.map(one, jobs))


def _compare_recorded(out, t, o, n, vcap, ctx):
    assert_result_equal(out.results[t], o.result, ctx)
    assert_records_equal(out.records[t], o.records, n, ctx)
    nv = int(o.result["evictions"])
    assert nv <= vcap, ctx
    gv = out.victims[t * vcap: t * vcap + nv]
    assert np.array_equal(gv, o.victims[:nv]), ctx + " victims"


def test_config2_bench_launch_sampled(kvr, oracle_mod):
    import bench
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator
    (L,) = bench.c2_plan(0, 1)
    sim = Simulator(L.W, bench.B_BLOCKS, pending_ring=L.ring)
    out = sim.run([DeviceTrace(t) for t in L.traces], L.keys, L.policies(), trial_trace=L.trial_trace)
    assert np.all(out.results["status"] == 0)
    assert np.all(out.results["queries"] == bench.C2_QUERIES)
    cfg = oracle_mod.OracleConfig(W=L.W, capacity_blocks=bench.B_BLOCKS, pending_ring=L.ring)
    picks = [int(np.nonzero((L.trial_trace == tr) & (L.evict == ev))[0][-1])
             for tr in range(3) for ev in (0, 1)]
    orc = _oracle_many(oracle_mod, [(cfg, L.traces[L.trial_trace[t]],
                                     oracle_mod.OraclePolicy(eviction=int(L.evict[t])),
                                     int(L.keys[t]), False, 0) for t in picks])
    for t, o in zip(picks, orc):
        assert_result_equal(out.results[t], o.result, f"config2 trial {t}")


def test_config3_drift_100k_prefix_per_router(kvr, oracle_mod):
    from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array
    tr = wl.drift(8192, 1_000_000, seed=0xC5, W=16).prefix(100_000)
    pols = [Policy(eviction=1, router=0),                                  # LBGR, App. A
            Policy(eviction=1, router=0, mu=0.992, delta_t_ms=10.0),       # collapsing cell
            Policy(eviction=1, router=1, w_load=0.25, w_hit=4.0),          # STATIC
            Policy(eviction=1, router=2, tau=2.0)]                         # THRESHOLD
    keys = [1, 1367, 2732, 4096]
    n, vcap = tr.n_queries, tr.total_blocks
    sim = Simulator(16, 512, pending_ring=n, record_trials=len(keys))
    out = sim.run(DeviceTrace(tr), np.array(keys, np.uint64), policies_array(pols),
                  victims_cap=vcap * len(keys))
    cfg = oracle_mod.OracleConfig(W=16, capacity_blocks=512, pending_ring=n)
    orc = _oracle_many(oracle_mod, [(cfg, tr, to_oracle_policy(oracle_mod, p), k, True, vcap)
                                    for p, k in zip(pols, keys)])
    for t, o in enumerate(orc):
        assert int(out.results[t]["status"]) == 0 and int(out.results[t]["queries"]) == n
        _compare_recorded(out, t, o, n, vcap, f"config3 trial {t} {pols[t]}")
    assert int(out.results[1]["max_pending"]) > 1000      # the deep-queue cell is exercised


@pytest.mark.parametrize("B", [64, 1024, 4096])
def test_config4_adversarial_full(kvr, oracle_mod, B):
    tr = wl.adv(B, 4, 8, seed=0xC6)
    pols = [kvr.Policy(eviction=0, router=3), kvr.Policy(eviction=1, router=3)]
    out, orc = compare(oracle_mod, kvr, tr, 1, B, pols, [3, 4], record=False)
    # Thm 1: in steady state L-LRU misses every tail -> one eviction per query
    # (the first cycle overflows by one block, then every query misses its tail)
    N = tr.n_queries
    assert int(out.results[0]["evictions"]) == N - B + 3
    assert int(out.results[1]["evictions"]) < int(out.results[0]["evictions"]) // 2


@pytest.mark.parametrize("W", [4, 8, 16, 32])
def test_config5_every_cell_recipe_size(kvr, oracle_mod, W):
    import bench
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator
    trs = bench.c5_traces(W)
    cell = bench.c5_cell_of(bench.C5_TRIALS)
    wi = bench.C5_WS.index(W)
    # the first trial of each of this W's 12 cells in the fixed 65,536 list (bench keys)
    tids = np.array([int(np.nonzero(cell == 12 * wi + c)[0][0]) for c in range(12)])
    ti = (cell[tids] % 12).astype(np.uint32)
    keys = (tids + 1).astype(np.uint64)
    evict = (keys % 2 == 0).astype(np.uint32)
    L = bench.Launch(W, trs, tids, ti, keys, evict)
    stride = max(t.n_queries for t in trs)
    vcap = max(t.total_blocks for t in trs)
    sim = Simulator(W, bench.B_BLOCKS, pending_ring=L.ring, record_trials=len(keys))
    out = sim.run([DeviceTrace(t) for t in trs], keys, L.policies(), trial_trace=ti,
                  victims_cap=vcap * len(keys))
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=bench.B_BLOCKS, pending_ring=L.ring)
    orc = _oracle_many(oracle_mod, [(cfg, trs[ti[t]], oracle_mod.OraclePolicy(eviction=int(evict[t])),
                                     int(keys[t]), True, vcap) for t in range(len(keys))])
    assert max(t.n_queries for t in trs) == 16384 and stride == 16384     # LD-high
    for t, o in enumerate(orc):
        n = trs[ti[t]].n_queries
        assert int(out.results[t]["status"]) == 0 and int(out.results[t]["queries"]) == n
        _compare_recorded(out, t, o, n, vcap, f"config5 W={W} cell {12 * wi + int(ti[t])} "
                                               f"({trs[ti[t]].name}) trial {tids[t]}")
    assert {int(e) for e in evict} == {0, 1}
