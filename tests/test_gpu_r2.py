"""GPU parity for the round-2 changes of the beta = 1 engine and the batching engine.

* pooled pending FIFOs (32-record chunks, per-worker free lists): deep queues that
  span many chunks, chunk reuse, and the per-worker cap `pending_ring` (overflow stop
  point) against the oracle's std::deque FIFOs;
* NaN score ordering (A37) and per-trial policy validation (KVR_TRIAL_BAD_POLICY for
  mu outside [0, 2), non-finite parameters) identical to the oracle's checks;
* KVR_TRIAL_BAD_TRACE for a trial -> trace index out of range (both kernels).
"""
import math

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


@pytest.mark.parametrize("force_tier", [1, 2])
def test_deep_fifo_chunks_parity(kvr, oracle_mod, force_tier):
    """Overloaded arrivals (util 3) and the collapsing NLMS step mu = 0.992: queues grow to
    hundreds of pending completions per worker (dozens of 32-record chunks), drain, and
    chunks are reused.  Every field, record and victim equals the oracle's."""
    tr = wl.gsp(30, 40, 0.5, seed=21, W=4, util=3.0, lengths=(128, 256, 512))
    pols = [kvr.Policy(eviction=e, mu=mu, router=r)
            for e, mu, r in ((1, 0.992, 0), (0, 0.992, 0), (1, 0.008, 0), (0, 0.0, 1), (1, 0.0, 2))]
    out, orc = compare(oracle_mod, kvr, tr, 4, 160, pols, [11, 12, 13, 14, 15],
                       ring=tr.n_queries, force_tier=force_tier)
    assert max(int(r["max_pending"]) for r in out.results) > 96     # > 3 chunks deep
    assert all(int(r["status"]) == 0 for r in out.results)


@pytest.mark.parametrize("ring", [1, 31, 32, 33, 70])
def test_fifo_cap_stop_point(kvr, oracle_mod, ring):
    """The per-worker cap pending_ring still stops a trial at the same query as the
    oracle (status 1 and the query count), at and around chunk boundaries."""
    tr = wl.gsp(20, 30, 0.5, seed=22, W=2, util=4.0, lengths=(128, 256))
    pols = [kvr.Policy(eviction=1, mu=0.992), kvr.Policy(eviction=0, router=2)]
    out, orc = compare(oracle_mod, kvr, tr, 2, 64, pols, [1, 2], ring=ring)
    assert any(o.result["status"] == 1 for o in orc)


def test_nan_score_ranks_last(kvr, oracle_mod):
    """P37 on the GPU: worker 0's score is inf - inf = NaN, worker 1's -inf -> i* = 1."""
    p = list(range(1, 126))
    tr = wl.from_paths([p, p + list(range(5000, 5125))], arrival_ms=[0.0, 0.0])
    pols = [kvr.Policy(eviction=0, mu=0.0, theta0=(1e308, -1e308, 0.0, 0.0))]
    out, orc = compare(oracle_mod, kvr, tr, 2, 512, pols, [0])
    assert list(out.records[0]["worker"][:2]) == [0, 1]


BAD = [dict(mu=2.0), dict(mu=-0.5), dict(mu=math.nan), dict(theta0=(math.inf, 0.0, 0.0, 0.0)),
       dict(w_load=math.nan), dict(est_alpha_cached_ms=math.inf), dict(tau=math.inf)]


@pytest.mark.parametrize("beta", [0, 2])
def test_per_trial_policy_validation(kvr, oracle_mod, beta):
    """Device-side checks of per-trial policies match the oracle's refusals (rc = 1):
    those trials get KVR_TRIAL_BAD_POLICY and do not run; valid ones are unaffected."""
    tr = wl.gsp(6, 5, 0.5, seed=23, W=2)
    good = kvr.Policy(eviction=1, mu=1.999, delta_t_ms=math.inf)
    pols = [kvr.Policy(eviction=1, **b) for b in BAD] + [good]
    sim = kvr.Simulator(2, 512, batch_slots=beta)
    out = sim.run(kvr.DeviceTrace(tr), np.arange(1, len(pols) + 1, dtype=np.uint64),
                  kvr.policies_array(pols))
    st = [int(r["status"]) for r in out.results]
    assert st[:-1] == [kvr.TRIAL_BAD_POLICY] * len(BAD)
    assert all(int(r["queries"]) == 0 for r in out.results[:-1])
    assert st[-1] == 0 and int(out.results[-1]["queries"]) == tr.n_queries
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=512, batch_slots=beta)
    for b in BAD:
        assert oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=1, **b), 1).rc == 1


@pytest.mark.parametrize("beta", [0, 2])
def test_trial_trace_out_of_range(kvr, beta):
    """kvr_sim_run_multi: a trial whose trace index is >= n_traces gets
    KVR_TRIAL_BAD_TRACE and does not run; the others are unaffected."""
    trs = [wl.gsp(5, 4, 0.5, seed=24, W=2), wl.gsp(5, 4, 0.9, seed=25, W=2)]
    sim = kvr.Simulator(2, 512, batch_slots=beta)
    dts = [kvr.DeviceTrace(t) for t in trs]
    out = sim.run(dts, np.array([1, 2, 3, 4], np.uint64), trial_trace=np.array([0, 2, 1, 64], np.uint32))
    st = [int(r["status"]) for r in out.results]
    assert st == [0, kvr.TRIAL_BAD_TRACE, 0, kvr.TRIAL_BAD_TRACE]
    assert [int(r["queries"]) for r in out.results] == [trs[0].n_queries, 0, trs[1].n_queries, 0]


def test_batching_deep_queue_counters(kvr, oracle_mod):
    """Batching engine with a long waiting FIFO (util 3, beta = 2): counters flushed as
    they grow still equal the oracle's sums."""
    tr = wl.gsp(30, 30, 0.5, seed=26, W=2, util=3.0, lengths=(128, 256))
    pols = [kvr.Policy(eviction=1), kvr.Policy(eviction=0, router=1)]
    compare_batched(oracle_mod, kvr, tr, 2, 64, 2, pols, [5, 6], ring=tr.n_queries)
