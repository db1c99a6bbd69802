"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): hit counts, routing and eviction decisions bit-exact
(per-query worker, hits, victims, digest); fp64 latency / TTFT / makespan aggregates
within 1e-12 relative — both sides evaluate the same expressions in the same order
without contraction, so the tests require exact equality.
"""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import compare, run_gpu, run_oracle, assert_result_equal

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


def _pols(kvr, **kw):
    return kvr.Policy(**kw)


# ------------------------------------------------------------------ packer (a0)
@pytest.mark.parametrize("maker", [
    lambda: wl.random_tree(200, 1, max_len=70, alphabet=3, max_out=2),
    lambda: wl.gsp(12, 7, 0.5, seed=3),
    lambda: wl.mt(9, 0.5, seed=4),
    lambda: wl.from_paths([[1]]),
])
def test_packer_chained_identities_bit_exact(kvr, oracle_mod, maker):
    tr = maker()
    from paper_2601_18999_b200.kvr import DeviceTrace
    dt = DeviceTrace(tr)
    assert np.array_equal(dt.chained_hashes(), oracle_mod.chain(tr))
    assert dt.max_path_blocks == tr.max_blocks and dt.n_queries == tr.n_queries


def test_packer_salt(kvr, oracle_mod):
    tr = wl.gsp(5, 4, 0.5, seed=1)
    tr.hash_salt = 0xDEADBEEF12345678
    from paper_2601_18999_b200.kvr import DeviceTrace
    assert np.array_equal(DeviceTrace(tr).chained_hashes(), oracle_mod.chain(tr))


@pytest.mark.parametrize("defect", ["arrival_decreasing", "arrival_nan", "n_in_zero", "offsets"])
def test_packer_rejects_malformed_trace(kvr, defect):
    from paper_2601_18999_b200.kvr import DeviceTrace, KvrError
    tr = wl.gsp(4, 4, 0.5, seed=2)
    if defect == "arrival_decreasing":
        tr.arrival_ms[5] = tr.arrival_ms[4] - 1.0
    elif defect == "arrival_nan":
        tr.arrival_ms[3] = np.nan
    elif defect == "n_in_zero":
        tr.n_in_blocks[2] = 0
    else:
        tr.block_offsets[3] += 1
    with pytest.raises(KvrError) as e:
        DeviceTrace(tr)
    assert e.value.status == 1


# --------------------------------------------------------------- replay (a1-a5)
POLICY_GRID = [
    dict(eviction=0, router=0), dict(eviction=1, router=0),
    dict(eviction=1, rlt_fallback=1, router=0), dict(eviction=1, rlt_fallback=2, router=0),
    dict(eviction=1, router=1, w_hit=2.0, w_load=0.5), dict(eviction=0, router=2, tau=1.25),
    dict(eviction=1, router=3), dict(eviction=1, router=4), dict(eviction=0, router=4),
    dict(eviction=1, router=0, mu=0.3, rho=0.5, delta_t_ms=7.0),
    dict(eviction=1, router=0, delta_t_ms=float("inf")),
]


@pytest.mark.parametrize("W,B", [(1, 6), (2, 9), (3, 16), (5, 12), (32, 8)])
def test_replay_small_random_all_policies(kvr, oracle_mod, W, B):
    """Ragged random prefix-sharing traces, every eviction x fallback x router."""
    tr = wl.random_tree(300, 10 + W, max_len=min(6, B - 1), alphabet=3, max_out=1, W=W)
    pols = [_pols(kvr, **g) for g in POLICY_GRID]
    keys = [1000 + 17 * i for i in range(len(pols))]
    compare(oracle_mod, kvr, tr, W, B, pols, keys, truth=(0.5, 1.0, 3.0), bins=32)


@pytest.mark.parametrize("force_tier", [1, 2])
def test_replay_tiers_agree(kvr, oracle_mod, force_tier):
    tr = wl.gsp(20, 12, 0.5, seed=7, W=4, lengths=(256, 512, 1024))
    pols = [_pols(kvr, eviction=e, rlt_fallback=f) for e, f in ((1, 0), (0, 0), (1, 1), (1, 2))]
    compare(oracle_mod, kvr, tr, 4, 160, pols, [3, 5, 7, 9], force_tier=force_tier)


def test_config1_bit_exact(kvr, oracle_mod):
    """BASELINE config 1: W=4, 1,000 GSP queries, B=512, 8 replays (LBGR; RLT x4, LRU x4),
    every trial recorded: digests, per-query (i*, h, victims), TTFT and latency arrays."""
    tr = wl.gsp(40, 25, 0.5, seed=0xC1, W=4)
    pols = [_pols(kvr, eviction=1 if t < 4 else 0) for t in range(8)]
    compare(oracle_mod, kvr, tr, 4, 512, pols, list(range(1, 9)), bins=64)


def test_multi_trace_launch(kvr, oracle_mod):
    trs = [wl.gsp(10, 8, r, seed=20 + i, W=3) for i, r in enumerate((0.3, 0.5, 0.9))]
    pols = [_pols(kvr, eviction=t % 2) for t in range(9)]
    keys = list(range(50, 59))
    tt = np.array([t % 3 for t in range(9)], dtype=np.uint32)
    out, _, _ = run_gpu(kvr, trs, 3, 256, pols, keys, (0.0, 1.0, 20.0), 256, True, 4096,
                        trial_trace=tt)
    for t in range(9):
        o = run_oracle(oracle_mod, trs[tt[t]], 3, 256, [pols[t]], [keys[t]], (0.0, 1.0, 20.0),
                       256, False, 0)[0]
        assert_result_equal(out.results[t], o.result, f"trial {t}")


def test_ring_overflow_status(kvr, oracle_mod):
    tr = wl.gsp(10, 10, 0.5, seed=1, rate_per_s=1000.0)     # overload: queues grow
    pols = [_pols(kvr, eviction=1, router=3), _pols(kvr, eviction=0, router=0)]
    out, orc = compare(oracle_mod, kvr, tr, 2, 300, pols, [1, 2], ring=4)
    assert all(int(r["status"]) == 1 for r in out.results)


def test_edge_cases(kvr, oracle_mod):
    pols = [_pols(kvr, eviction=e) for e in (0, 1)]
    # B = 1 with single-block paths, W = 1
    tr = wl.from_paths([[k % 3] for k in range(40)], arrival_ms=np.arange(40) * 100.0)
    compare(oracle_mod, kvr, tr, 1, 1, pols, [1, 2])
    # paths exactly B long, all arrivals equal
    tr = wl.from_paths([[1, 2, 3, 4], [1, 2, 5, 6], [7, 8, 9, 10], [1, 2, 3, 4]])
    compare(oracle_mod, kvr, tr, 2, 4, pols, [3, 4])
    # long paths (several 32-block windows + ragged tail) with outputs
    tr = wl.random_tree(60, 5, max_len=100, alphabet=2, max_out=3, W=2)
    compare(oracle_mod, kvr, tr, 2, 130, pols, [5, 6])


def test_empty_trace(kvr):
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator
    tr = wl.from_paths([])
    dt = DeviceTrace(tr)
    sim = Simulator(2, 8)
    out = sim.run(dt, np.array([1, 2], np.uint64))
    assert np.all(out.results["queries"] == 0) and np.all(out.results["status"] == 0)
    assert np.all(out.results["decision_digest"] == np.array([1, 2], np.uint64))


def test_capacity_precondition(kvr):
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, KvrError
    tr = wl.from_paths([[1, 2, 3, 4, 5]])
    sim = Simulator(1, 4)
    with pytest.raises(KvrError) as e:
        sim.run(DeviceTrace(tr), np.array([1], np.uint64))
    assert e.value.status == 2


def test_determinism_and_launch_invariance(kvr):
    """P20: identical inputs -> identical bytes; a trial's result does not depend on
    which launch or position runs it (the basis of multi-GPU sharding)."""
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, policies_array, Policy
    tr = wl.gsp(30, 10, 0.5, seed=9, W=8)
    dt = DeviceTrace(tr)
    sim = Simulator(8, 512)
    keys = np.arange(1, 65, dtype=np.uint64)
    pols = policies_array([Policy(eviction=int(k) % 2) for k in keys])
    a = sim.run(dt, keys, pols).results
    b = sim.run(dt, keys, pols).results
    assert a.tobytes() == b.tobytes()
    c = sim.run(dt, keys[1::2], pols[1::2]).results
    assert c.tobytes() == a[1::2].tobytes()


def test_adversarial_large_B_global_tier(kvr, oracle_mod):
    """Config 4 family at B = 65,536 (global-memory tier, u32 slot ids), sampled queries."""
    B = 65536
    tr = wl.adv(B, 4, 2).prefix(66000)
    pols = [_pols(kvr, eviction=0, router=3), _pols(kvr, eviction=1, router=3)]
    compare(oracle_mod, kvr, tr, 1, B, pols, [1, 2], record=False)


def test_identity_digest(kvr, oracle_mod):
    """The multi-GPU trace checksum (bench.py reduce): same raw trace -> same digest on
    every load; a different salt (different identities) -> a different digest."""
    from paper_2601_18999_b200.kvr import DeviceTrace
    tr = wl.gsp(6, 5, 0.5, seed=3)
    a, b = DeviceTrace(tr).identity_digest(), DeviceTrace(tr).identity_digest()
    assert a == b and a != 0
    tr.hash_salt = 99
    assert DeviceTrace(tr).identity_digest() != a


def test_collision_check(kvr, oracle_mod):
    """kvr_trace_check_collisions (device sort + adjacent compare) vs the oracle's
    count on a crafted genuine collision, after re-salting, and on normal traces."""
    from collision_util import colliding_pair
    from paper_2601_18999_b200.kvr import (DeviceTrace, ERR_HASH_COLLISION, kvr_trace_check_collisions,
                                           kvr_trace_collision_bytes)
    import torch
    b2 = colliding_pair(11, 12, 13)
    tr = wl.from_paths([[11, 12], [13, b2], [11, 12, 5]], n_out=[0, 0, 1])
    dt = DeviceTrace(tr)
    scratch = torch.empty(kvr_trace_collision_bytes(dt.handle), dtype=torch.uint8, device="cuda")
    st, n = kvr_trace_check_collisions(dt.handle, dt.keys, scratch)
    assert st == ERR_HASH_COLLISION and n == oracle_mod.count_collisions(tr) == 2
    tr.hash_salt = 77
    assert DeviceTrace(tr).collisions() == oracle_mod.count_collisions(tr) == 0
    for t in (wl.gsp(40, 30, 0.5, seed=1), wl.mt(24, 0.9, seed=2), wl.from_paths([[1]]),
              wl.from_paths([])):
        assert DeviceTrace(t).collisions() == 0


def test_fuzz_random_configs(kvr, oracle_mod):
    """150 random (W, B, trace, policy, ring, tier, histogram) draws of the beta = 1
    kernel, 3 trials each incl. the extended policies (LBGR_RLS, tracker bias)."""
    rng = np.random.default_rng(7)
    for it in range(150):
        W = int(rng.integers(1, 12))
        tr = wl.random_tree(int(rng.integers(20, 150)), 3000 + it, max_len=int(rng.integers(2, 9)),
                            alphabet=int(rng.integers(2, 4)), max_out=int(rng.integers(0, 3)), W=W,
                            util=float(rng.uniform(0.3, 3.0)))
        B = int(tr.max_blocks) + int(rng.integers(0, 12))
        pols = []
        for _ in range(3):
            pols.append(kvr.Policy(eviction=int(rng.integers(0, 2)), rlt_fallback=int(rng.integers(0, 3)),
                                   router=int(rng.integers(0, 6)), tau=float(rng.uniform(1.0, 3.0)),
                                   w_hit=float(rng.uniform(0, 2)), w_load=float(rng.uniform(0, 2)),
                                   mu=float(rng.uniform(0.05, 1.0)), rho=float(rng.uniform(0.5, 1.0)),
                                   delta_t_ms=float(rng.uniform(5, 50)),
                                   tracker_lag=int(rng.integers(0, 2)),
                                   tracker_grain=int(rng.integers(1, 4))))
        keys = [int(k) for k in rng.integers(1, 1 << 40, size=3)]
        compare(oracle_mod, kvr, tr, W, B, pols, keys,
                truth=(float(rng.uniform(0, 0.5)), 1.0, float(rng.uniform(0, 5))),
                ring=int(rng.integers(4, 64)), force_tier=int(rng.integers(1, 3)),
                bins=int(rng.integers(0, 2)) * 32)


def test_fuzz_larger_caches(kvr, oracle_mod):
    """Random GSP / multi-turn / long-document traces at B in [64, 2048] (crossing the
    1,024-slot register-bitmap / deferred-apply limit) and W in [1, 16], both tiers."""
    rng = np.random.default_rng(11)
    for it in range(24):
        W = int(rng.integers(1, 17))
        kind = it % 3
        if kind == 0:
            tr = wl.gsp(int(rng.integers(4, 12)), int(rng.integers(3, 10)), float(rng.uniform(0.2, 0.9)),
                        seed=100 + it, W=W, lengths=(128, 256, 512, 1024))
        elif kind == 1:
            tr = wl.mt(int(rng.integers(4, 16)), float(rng.uniform(0.2, 0.9)), seed=200 + it, W=W,
                       user_blocks=int(rng.integers(2, 8)))
        else:
            tr = wl.ld(int(rng.integers(4, 12)), int(rng.integers(2, 6)), seed=300 + it, W=W,
                       lengths=(256, 512, 1024))
        B = max(int(tr.max_blocks), int(rng.integers(64, 2049)))
        pols = [kvr.Policy(eviction=int(rng.integers(0, 2)), rlt_fallback=int(rng.integers(0, 3)),
                           router=int(rng.integers(0, 6))) for _ in range(2)]
        keys = [int(k) for k in rng.integers(1, 1 << 40, size=2)]
        compare(oracle_mod, kvr, tr, W, B, pols, keys, force_tier=int(rng.integers(0, 3)))
