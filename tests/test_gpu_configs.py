"""GPU parity at BASELINE.json sizes (sampled where the oracle cannot finish).

* config 2: the exact launch bench.py times (3 x 100k-query traces, W=8, B=512,
  1,024 trials in one kvr_sim_run_multi); sampled trials are replayed by the
  oracle over the full 100k queries and compared field by field.
* config 3: DRIFT trace, W=16, LBGR / STATIC / THRESHOLD: oracle on a prefix.
* config 4: Thm 1 adversarial family, W=1, B in {64, 1024, 4096} full length.
* config 5 shapes: multi-turn and long-document traces at W=4 and W=32
  (W=32 runs the global-memory tier).
"""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import assert_result_equal, compare, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvr():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr as k
    return k


def test_config2_bench_launch_sampled(kvr, oracle_mod):
    import bench
    from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array
    trs = bench.build_traces()
    t_of, ev, keys = bench.trial_plan(0)
    sim = Simulator(bench.W_WORKERS, bench.B_BLOCKS, pending_ring=bench.RING)
    out = sim.run([DeviceTrace(t) for t in trs], keys,
                  policies_array([Policy(eviction=int(e)) for e in ev]), trial_trace=t_of)
    assert np.all(out.results["status"] == 0)
    assert np.all(out.results["queries"] == bench.N_QUERIES)
    cfg = oracle_mod.OracleConfig(W=bench.W_WORKERS, capacity_blocks=bench.B_BLOCKS,
                                  pending_ring=bench.RING)
    for t in (0, 400, 700, 1023):      # RLT r=0.3, RLT r=0.9, LRU r=0.5, LRU r=0.9 (last)
        o = oracle_mod.run(cfg, trs[t_of[t]], oracle_mod.OraclePolicy(eviction=int(ev[t])),
                           int(keys[t]))
        assert o.rc == 0
        assert_result_equal(out.results[t], o.result, f"config2 trial {t}")


@pytest.mark.parametrize("router,extra", [(0, {}), (1, dict(w_hit=4.0, w_load=0.25)),
                                          (2, dict(tau=2.0))])
def test_config3_drift_prefix(kvr, oracle_mod, router, extra):
    tr = wl.drift(8192, 1_000_000, seed=0xC5, W=16).prefix(12_000)
    pols = [kvr.Policy(eviction=1, router=router, **extra),
            kvr.Policy(eviction=1, router=router, mu=0.1, delta_t_ms=40.0, **extra)]
    compare(oracle_mod, kvr, tr, 16, 512, pols, [11, 12], record=True)


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


@pytest.mark.parametrize("W", [4, 32])
def test_config5_shapes(kvr, oracle_mod, W):
    B = 512
    for tr in (wl.mt(24, 0.5, seed=0xC7, W=W), wl.ld(32, 8, seed=0xC8, W=W),
               wl.gsp(24, 10, 0.9, seed=0xC9, W=W)):
        pols = [kvr.Policy(eviction=1), kvr.Policy(eviction=0)]
        compare(oracle_mod, kvr, tr, W, B, pols, [5, 6], record=True)
