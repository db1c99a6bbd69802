"""GPU parity of the continuous-batching kernel (kvr_batch.cu; SURVEY §8f #2,
DESIGN.md A30-A36) against the oracle's batching engine: decisions, hits,
victims, digests bit-exact; fp64 aggregates bit-equal (same per-worker order)."""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import compare_batched

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


GRID = [
    dict(eviction=0, router=0), dict(eviction=1, router=0),
    dict(eviction=1, rlt_fallback=1, router=0), dict(eviction=1, rlt_fallback=2, router=0),
    dict(eviction=1, router=1, w_hit=2.0, w_load=0.5), dict(eviction=0, router=2, tau=1.25),
    dict(eviction=1, router=3), dict(eviction=1, router=4), dict(eviction=0, router=5),
    dict(eviction=1, router=0, mu=0.3, rho=0.5, delta_t_ms=7.0),
]


def test_hand_example_p25(kvr, oracle_mod):
    tr = wl.from_paths([[1, 2], [1, 3], [4, 5], [1, 2]], arrival_ms=[0.0, 0.5, 1.0, 2.5],
                       block_tokens=1)
    pols = [kvr.Policy(eviction=e, router=3) for e in (0, 1)]
    out, orc = compare_batched(oracle_mod, kvr, tr, 1, 4, 2, pols, [0, 1], truth=(0.0, 1.0, 0.0))
    assert list(out.records[0]["latency_ms"][:4]) == [2.0, 1.0, 2.5, 0.0]


@pytest.mark.parametrize("W,beta", [(1, 1), (1, 3), (2, 2), (3, 1), (4, 4), (8, 2), (32, 2)])
def test_random_trees_all_policies(kvr, oracle_mod, W, beta):
    tr = wl.random_tree(250, 40 + W + beta, max_len=6, alphabet=3, max_out=1, W=W, util=1.3)
    B = beta * int(tr.max_blocks) + (W % 3)        # at or near the premise's tightest cache
    pols = [kvr.Policy(**g) for g in GRID]
    keys = [500 + 13 * i for i in range(len(pols))]
    compare_batched(oracle_mod, kvr, tr, W, B, beta, pols, keys, truth=(0.5, 1.0, 3.0), bins=32)


@pytest.mark.parametrize("force_tier", [1, 2])
def test_gsp_tiers(kvr, oracle_mod, force_tier):
    tr = wl.gsp(20, 12, 0.5, seed=7, W=4, lengths=(256, 512, 1024))
    beta = 2
    pols = [kvr.Policy(eviction=e, rlt_fallback=f) for e, f in ((1, 0), (0, 0), (1, 1), (1, 2))]
    compare_batched(oracle_mod, kvr, tr, 4, 160, beta, pols, [3, 5, 7, 9], force_tier=force_tier)


def test_long_paths_ragged(kvr, oracle_mod):
    """several 32-block windows + ragged tails, outputs, beta = 3"""
    tr = wl.random_tree(80, 5, max_len=70, alphabet=2, max_out=3, W=2, util=2.0)
    pols = [kvr.Policy(eviction=e) for e in (0, 1)] + [kvr.Policy(eviction=1, router=5)]
    compare_batched(oracle_mod, kvr, tr, 2, 3 * int(tr.max_blocks), 3, pols, [5, 6, 7])


def test_thm2_construction(kvr, oracle_mod):
    """Thm 2 lower-bound family through the GPU: L-LRU misses every
    rotating request (one eviction each in steady state)."""
    B, L, beta, cycles = 16, 4, 3, 10
    R = B - L - beta + 3
    prefix = [7000 + d for d in range(L - 1)]
    paths, arr = [], []
    t = 0.0
    for _ in range(cycles):
        for u in range(1, R + 1):
            for g in list(range(1, beta)) + [u + beta - 1]:
                paths.append(prefix + [9000 + g])
                arr.append(t)
            t += 1.0e5
    tr = wl.from_paths(paths, arrival_ms=arr)
    pols = [kvr.Policy(eviction=0, router=3), kvr.Policy(eviction=1, router=3)]
    out, orc = compare_batched(oracle_mod, kvr, tr, 1, B, beta, pols, [1, 2], truth=(0.0, 1.0, 0.0))
    # cold start fills B - (L - 1) = 13 tail slots; every later rotating request evicts once
    assert int(out.results[0]["evictions"]) == cycles * R - (B - L + 1 - (beta - 1))


def test_config_shapes_full(kvr, oracle_mod):
    """config-2 GSP shape (W = 8, B = 512, beta = 3 = the largest with 3*129 <= 512) and
    config-5 multi-turn / long-doc shapes; full traces, sampled trials."""
    for tr, W, beta, B in ((wl.gsp(125, 40, 0.5, seed=0xC3, W=8, lengths=(256, 512, 1024, 2048)), 8, 3, 512),
                           (wl.mt(24, 0.5, seed=0xC7, W=4), 4, 1, 512),
                           (wl.ld(32, 8, seed=0xC8, W=4), 4, 2, 1024)):
        pols = [kvr.Policy(eviction=1), kvr.Policy(eviction=0), kvr.Policy(eviction=1, router=1)]
        compare_batched(oracle_mod, kvr, tr, W, B, beta, pols, [5, 6, 7], record=True)


def test_ring_overflow_and_validation(kvr, oracle_mod):
    from paper_2601_18999_b200.kvr import DeviceTrace, KvrError, Simulator
    tr = wl.gsp(10, 10, 0.5, seed=1, rate_per_s=1000.0)     # overload: queues grow
    pols = [kvr.Policy(eviction=1, router=3), kvr.Policy(eviction=0, router=0)]
    out, _ = compare_batched(oracle_mod, kvr, tr, 2, 300, 1, pols, [1, 2], ring=4)
    assert all(int(r["status"]) == 1 for r in out.results)
    # premise beta * L_max <= B
    sim = Simulator(1, 7, batch_slots=2)
    with pytest.raises(KvrError) as e:
        sim.run(DeviceTrace(wl.from_paths([[1, 2, 3, 4]])), np.array([1], np.uint64))
    assert e.value.status == 2
    # OPT / tracker bias are beta = 1 analyses (A36)
    with pytest.raises(KvrError):
        Simulator(1, 8, policy=kvr.Policy(eviction=2), batch_slots=2)
    with pytest.raises(KvrError):
        Simulator(2, 8, policy=kvr.Policy(tracker_grain=4), batch_slots=2)
    sim = Simulator(2, 128, batch_slots=2)
    from paper_2601_18999_b200.kvr import policies_array
    r = sim.run(DeviceTrace(wl.gsp(3, 3, 0.5, seed=2)), np.array([1, 2], np.uint64),
                policies_array([kvr.Policy(tracker_lag=1), kvr.Policy()])).results
    assert int(r[0]["status"]) == 3 and int(r[1]["status"]) == 0


def test_beta_sweep_multiserver_monotone(kvr, oracle_mod):
    """No shared blocks (every query misses everything), so service times do not
    depend on the cache: with the same arrivals and round-robin routing, FIFO start
    times are nonincreasing in the number of servers beta (Kiefer-Wolfowitz), hence
    every query's latency is too; each beta is also checked against the oracle."""
    rng = np.random.default_rng(3)
    N = 400
    lens = rng.integers(1, 9, size=N)
    paths, k = [], 1
    for n in lens:
        paths.append(list(range(k, k + int(n))))
        k += int(n)
    arr = np.cumsum(rng.exponential(40.0, size=N))
    tr = wl.from_paths(paths, arrival_ms=arr, out_tokens=[4] * N)
    prev = None
    for beta in (1, 2, 4, 8):
        out, _ = compare_batched(oracle_mod, kvr, tr, 4, 8 * 8, beta,
                                 [kvr.Policy(router=3, eviction=0)], [1], truth=(0.0, 1.0, 20.0))
        lat = out.records[0]["latency_ms"][:N].copy()
        assert int(out.results[0]["hit_tokens"]) == 0
        if prev is not None:
            assert np.all(lat <= prev)
        prev = lat


def test_config2_full_trace_sampled(kvr, oracle_mod):
    """The bench's full 100k-query config-2 trace (r = 0.5) through the batching kernel at
    the largest beta the premise allows at B = 512 (beta = 3, L_max = 129), in one launch of
    64 trials; two sampled trials (RLT, L-LRU) replayed by the oracle over all 100k queries."""
    import bench
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, policies_array
    from parity_util import BATCH_SUM_FIELDS, assert_result_equal
    tr = bench.c2_traces()[1]
    sim = Simulator(bench.C2_W, bench.B_BLOCKS, pending_ring=16384, batch_slots=3)
    keys = np.arange(1, 65, dtype=np.uint64)
    pols = [kvr.Policy(eviction=int(k) % 2) for k in keys]
    out = sim.run(DeviceTrace(tr), keys, policies_array(pols))
    assert np.all(out.results["status"] == 0)
    assert np.all(out.results["queries"] == tr.n_queries)
    cfg = oracle_mod.OracleConfig(W=bench.C2_W, capacity_blocks=bench.B_BLOCKS,
                                  pending_ring=16384, batch_slots=3)
    for t in (0, 63):
        o = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=int(keys[t]) % 2), int(keys[t]))
        assert o.rc == 0
        assert_result_equal(out.results[t], o.result, f"batching config2 trial {t}",
                            rel_fields=BATCH_SUM_FIELDS)


def test_edge_cases(kvr, oracle_mod):
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator
    pols = [kvr.Policy(eviction=e) for e in (0, 1)] + [kvr.Policy(eviction=1, rlt_fallback=1)]
    # B = 1, beta = 1, single-block paths, W = 1
    tr = wl.from_paths([[k % 3] for k in range(40)], arrival_ms=np.arange(40) * 100.0)
    compare_batched(oracle_mod, kvr, tr, 1, 1, 1, pols, [1, 2, 3])
    # beta = 64 (the maximum) with single-block paths, everything arriving at once
    tr = wl.from_paths([[k % 70] for k in range(300)])
    compare_batched(oracle_mod, kvr, tr, 2, 64, 64, pols, [4, 5, 6])
    # W = 32, both tiers
    tr = wl.random_tree(200, 77, max_len=4, alphabet=3, max_out=1, W=32, util=2.0)
    for ft in (1, 2):
        compare_batched(oracle_mod, kvr, tr, 32, 2 * int(tr.max_blocks), 2, pols, [7, 8, 9],
                        force_tier=ft)
    # empty trace
    sim = Simulator(2, 8, batch_slots=2)
    out = sim.run(DeviceTrace(wl.from_paths([])), np.array([1, 2], np.uint64))
    assert np.all(out.results["queries"] == 0) and np.all(out.results["status"] == 0)
    assert np.all(out.results["decision_digest"] == np.array([1, 2], np.uint64))


def test_multi_trace_launch(kvr, oracle_mod):
    """kvr_sim_run_multi with the batching kernel: trials over three traces in one launch."""
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, policies_array
    from parity_util import BATCH_SUM_FIELDS, assert_result_equal
    trs = [wl.gsp(10, 8, r, seed=20 + i, W=3, lengths=(256, 512)) for i, r in enumerate((0.3, 0.5, 0.9))]
    pols = [kvr.Policy(eviction=t % 2, router=(0, 1, 5)[t % 3]) for t in range(9)]
    keys = np.arange(50, 59, dtype=np.uint64)
    tt = np.array([t % 3 for t in range(9)], dtype=np.uint32)
    sim = Simulator(3, 128, batch_slots=2)
    out = sim.run([DeviceTrace(t) for t in trs], keys, policies_array(pols), trial_trace=tt)
    cfg = oracle_mod.OracleConfig(W=3, capacity_blocks=128, batch_slots=2)
    from parity_util import to_oracle_policy
    for t in range(9):
        o = oracle_mod.run(cfg, trs[tt[t]], to_oracle_policy(oracle_mod, pols[t]), int(keys[t]))
        assert o.rc == 0
        assert_result_equal(out.results[t], o.result, f"trial {t}", rel_fields=BATCH_SUM_FIELDS)


def test_fuzz_random_configs(kvr, oracle_mod):
    """150 random (W, beta, B, trace, policy, ring, tier) draws, 3 trials each, bit-exact."""
    rng = np.random.default_rng(2024)
    for it in range(150):
        W = int(rng.integers(1, 9))
        beta = int(rng.integers(1, 5))
        tr = wl.random_tree(int(rng.integers(20, 120)), 900 + it, max_len=int(rng.integers(2, 9)),
                            alphabet=int(rng.integers(2, 4)), max_out=int(rng.integers(0, 3)), W=W,
                            util=float(rng.uniform(0.3, 3.0)))
        B = beta * int(tr.max_blocks) + int(rng.integers(0, 6))
        pols = []
        for _ in range(3):
            pols.append(kvr.Policy(eviction=int(rng.integers(0, 2)), rlt_fallback=int(rng.integers(0, 3)),
                                   router=int(rng.integers(0, 6)), tau=float(rng.uniform(1.0, 3.0)),
                                   w_hit=float(rng.uniform(0, 2)), w_load=float(rng.uniform(0, 2)),
                                   mu=float(rng.uniform(0.05, 1.0)), rho=float(rng.uniform(0.5, 1.0)),
                                   delta_t_ms=float(rng.uniform(5, 50))))
        keys = [int(k) for k in rng.integers(1, 1 << 40, size=3)]
        compare_batched(oracle_mod, kvr, tr, W, B, beta, pols, keys,
                        truth=(float(rng.uniform(0, 0.5)), 1.0, float(rng.uniform(0, 5))),
                        ring=int(rng.integers(4, 64)), force_tier=int(rng.integers(1, 3)))


def test_fuzz_larger_caches(kvr, oracle_mod):
    """Batching kernel on random GSP / multi-turn / long-document traces, B up to 2048."""
    rng = np.random.default_rng(13)
    for it in range(18):
        W = int(rng.integers(1, 17))
        beta = int(rng.integers(1, 4))
        kind = it % 3
        if kind == 0:
            tr = wl.gsp(int(rng.integers(4, 12)), int(rng.integers(3, 10)), float(rng.uniform(0.2, 0.9)),
                        seed=400 + it, W=W, lengths=(128, 256, 512), util=2.0)
        elif kind == 1:
            tr = wl.mt(int(rng.integers(4, 16)), float(rng.uniform(0.2, 0.9)), seed=500 + it, W=W,
                       user_blocks=int(rng.integers(2, 8)), util=2.0)
        else:
            tr = wl.ld(int(rng.integers(4, 12)), int(rng.integers(2, 6)), seed=600 + it, W=W,
                       lengths=(256, 512), util=2.0)
        B = max(beta * int(tr.max_blocks), int(rng.integers(64, 2049)))
        pols = [kvr.Policy(eviction=int(rng.integers(0, 2)), rlt_fallback=int(rng.integers(0, 3)),
                           router=int(rng.integers(0, 6))) for _ in range(2)]
        keys = [int(k) for k in rng.integers(1, 1 << 40, size=2)]
        compare_batched(oracle_mod, kvr, tr, W, B, beta, pols, keys)
