"""Offline Belady OPT on the GPU (OPT = evict the leaf whose next use
is furthest): the device next-use index, and OPT replays at W = 1
compared field by field with the oracle's full replay (kvro_run, W = 1, OPT, pinned
to the exhaustive minimum by test_p10b)."""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import compare

pytestmark = pytest.mark.gpu

INF = 0xFFFFFFFF


@pytest.fixture(scope="module")
def kvr():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr as k
    return k


def expected_next_use(oracle_mod, tr):
    """Backward scan over the ORACLE's chained identities (no GPU input)."""
    H = oracle_mod.chain(tr)
    off = np.asarray(tr.block_offsets, dtype=np.int64)
    nu = np.full(len(H), INF, dtype=np.uint32)
    last = {}
    for j in range(tr.n_queries - 1, -1, -1):
        for o in range(off[j], off[j + 1]):
            nu[o] = last.get(int(H[o]), INF)
        for o in range(off[j], off[j + 1]):
            last[int(H[o])] = j
    return nu


@pytest.mark.parametrize("make", [
    lambda: wl.gsp(20, 12, 0.5, seed=0x51, W=4),
    lambda: wl.adv(64, 4, 4, seed=0x52),
    lambda: wl.random_tree(300, 0x53, max_len=6, alphabet=3, max_out=2),
    lambda: wl.mt(16, 0.5, seed=0x54, W=4),
])
def test_next_use_index(kvr, oracle_mod, make):
    tr = make()
    dt = kvr.DeviceTrace(tr).with_next_use()
    assert np.array_equal(dt.next_use(), expected_next_use(oracle_mod, tr))


def test_next_use_empty_trace(kvr):
    dt = kvr.DeviceTrace(wl.from_paths([])).with_next_use()
    assert dt.n_blocks_total == 0


@pytest.mark.parametrize("tier", [1, 2])
def test_opt_parity_small(kvr, oracle_mod, tier):
    for seed in range(6):
        tr = wl.random_tree(400, 0x60 + seed, max_len=8, alphabet=3, max_out=2)
        for B in (8, 16, 40):
            if tr.max_blocks > B:
                continue
            pols = [kvr.Policy(eviction=kvr.EVICT_OPT, router=r) for r in (0, 3)]
            compare(oracle_mod, kvr, tr, 1, B, pols, [1, 2], record=True, force_tier=tier,
                    next_use=True)


def test_opt_parity_workloads(kvr, oracle_mod):
    for tr in (wl.gsp(24, 10, 0.9, seed=0x71, W=1), wl.mt(24, 0.5, seed=0x72, W=1),
               wl.ld(24, 8, seed=0x73, W=1)):
        pols = [kvr.Policy(eviction=kvr.EVICT_OPT)]
        compare(oracle_mod, kvr, tr, 1, 512, pols, [9], record=True, next_use=True)


@pytest.mark.parametrize("B", [64, 1024, 4096])
def test_config4_opt_thm1(kvr, oracle_mod, B):
    """Thm 1 family at config 4 capacities: OPT matches the oracle over
    the full trace; L-LRU misses every tail while OPT misses about once per phase of
    B-L+2 queries (the oracle pins the exact per-phase counts, P6/P7)."""
    L, cycles = 4, 8
    tr = wl.adv(B, L, cycles, seed=0xC6)
    pols = [kvr.Policy(eviction=kvr.EVICT_OPT, router=3), kvr.Policy(eviction=kvr.EVICT_LRU, router=3)]
    out, _ = compare(oracle_mod, kvr, tr, 1, B, pols, [3, 4], record=False, next_use=True)
    opt_ev, lru_ev = int(out.results[0]["evictions"]), int(out.results[1]["evictions"])
    assert lru_ev == tr.n_queries - B + 3
    # OPT: about one eviction per cycle; L-LRU: every tail after the cold first cycle
    assert 0 < opt_ev <= cycles + 1 and lru_ev >= (cycles - 1) * (B - L + 1)


def test_opt_policy_validation(kvr):
    tr = wl.adv(16, 4, 2, seed=1)
    with pytest.raises(kvr.KvrError):     # OPT is defined for one cache
        kvr.Simulator(2, 16, policy=kvr.Policy(eviction=kvr.EVICT_OPT))
    sim = kvr.Simulator(1, 16, policy=kvr.Policy(eviction=kvr.EVICT_OPT))
    with pytest.raises(kvr.KvrError):     # no next-use index on the trace
        sim.run(kvr.DeviceTrace(tr), np.array([1], np.uint64))
    # per-trial OPT policy at W = 2 (or without an index): that trial alone is refused
    sim2 = kvr.Simulator(2, 16)
    out = sim2.run(kvr.DeviceTrace(tr).with_next_use(), np.array([1, 2], np.uint64),
                   kvr.policies_array([kvr.Policy(eviction=kvr.EVICT_OPT), kvr.Policy()]))
    assert int(out.results[0]["status"]) == 3 and int(out.results[1]["status"]) == 0
