"""Router variants on the GPU: LBGR with the RLS reading of the
0.992 update (router 5, reading A8b) against the oracle's full replay, field by
field and per query (decisions bit-exact; the RLS algebra runs in the oracle's
order).  The oracle's RLS step is pinned to closed-form weighted least squares
(test_p23)."""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl
from parity_util import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kvr():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2601_18999_b200 import build
    build.build()
    from paper_2601_18999_b200 import kvr as k
    return k


@pytest.mark.parametrize("W", [1, 4, 8])
def test_lbgr_rls_parity(kvr, oracle_mod, W):
    tr = wl.gsp(30, 16, 0.5, seed=0x81 + W, W=W)
    pols = [kvr.Policy(router=kvr.ROUTE_LBGR_RLS, eviction=e, mu=mu, rls_p0=p0)
            for e, mu, p0 in ((1, 0.992, 1000.0), (0, 0.992, 10.0), (1, 0.9, 1e4), (1, 1.0, 1.0))]
    compare(oracle_mod, kvr, tr, W, 512, pols, [11, 12, 13, 14], record=True)


def test_lbgr_rls_drift_and_tiers(kvr, oracle_mod):
    tr = wl.drift(2048, 200_000, seed=0xC5, W=16).prefix(3000)
    for tier in (1, 2):
        pols = [kvr.Policy(router=kvr.ROUTE_LBGR_RLS), kvr.Policy(router=kvr.ROUTE_LBGR)]
        compare(oracle_mod, kvr, tr, 16, 512, pols, [21, 22], record=True, force_tier=tier)


def test_lbgr_rls_validation(kvr):
    with pytest.raises(kvr.KvrError):
        kvr.Simulator(4, 64, policy=kvr.Policy(router=kvr.ROUTE_LBGR_RLS, rls_p0=0.0))
    tr = wl.gsp(4, 4, 0.5, seed=1, W=2)
    sim = kvr.Simulator(2, 512)
    out = sim.run(kvr.DeviceTrace(tr), np.array([1, 2], np.uint64),
                  kvr.policies_array([kvr.Policy(router=kvr.ROUTE_LBGR_RLS, mu=1.5),
                                      kvr.Policy(router=kvr.ROUTE_LBGR_RLS)]))
    assert int(out.results[0]["status"]) == 3 and int(out.results[1]["status"]) == 0


@pytest.mark.parametrize("W", [2, 4, 8])
def test_tracker_parity(kvr, oracle_mod, W):
    """Approximate / stale global tracker (App. E, reading A29): the
    router scores with h~ (1-event lag and/or whole grains) while Eq. 1 uses h."""
    tr = wl.gsp(24, 12, 0.5, seed=0x90 + W, W=W)
    pols = []
    for router in (kvr.ROUTE_LBGR, kvr.ROUTE_STATIC_LINEAR, kvr.ROUTE_THRESHOLD):
        for lag, grain in ((1, 1), (0, 4), (1, 8)):
            pols.append(kvr.Policy(router=router, tracker_lag=lag, tracker_grain=grain,
                                   eviction=1 if grain != 4 else 0))
    compare(oracle_mod, kvr, tr, W, 512, pols, list(range(31, 31 + len(pols))), record=True)


def test_tracker_lag_hand_example(kvr, oracle_mod):
    tr = wl.from_paths([[11, 12, 13], [11, 12, 13]])
    pol = dict(router=kvr.ROUTE_STATIC_LINEAR, w_hit=1.0, w_load=1.0, eviction=0)
    out, _ = compare(oracle_mod, kvr, tr, 2, 8, [kvr.Policy(**pol), kvr.Policy(tracker_lag=1, **pol)],
                     [5, 5], record=True)
    assert list(out.records[0]["worker"][:2]) == [0, 0] and list(out.records[1]["worker"][:2]) == [0, 1]


def test_tracker_validation(kvr, oracle_mod):
    """A lag above KVR_MAX_TRACKER_LAG (32) is refused (host: KvrError; per trial: status
    3); a lag at a large capacity (B = 2048, the global-memory tier) runs and matches."""
    with pytest.raises(kvr.KvrError):
        kvr.Simulator(2, 64, policy=kvr.Policy(tracker_lag=33))
    with pytest.raises(kvr.KvrError):
        kvr.Simulator(2, 64, policy=kvr.Policy(tracker_grain=0))
    tr = wl.adv(2048, 4, 1, seed=2)
    sim = kvr.Simulator(1, 2048)
    out = sim.run(kvr.DeviceTrace(tr), np.array([1, 2], np.uint64),
                  kvr.policies_array([kvr.Policy(tracker_lag=33), kvr.Policy()]))
    assert int(out.results[0]["status"]) == 3 and int(out.results[1]["status"]) == 0
    tr = wl.gsp(10, 8, 0.5, seed=7, W=2, lengths=(128, 256))
    compare(oracle_mod, kvr, tr, 2, 2048, [kvr.Policy(tracker_lag=3, eviction=e) for e in (0, 1)],
            [1, 2], record=True)


def test_lean_kernel_refuses_extended_policies(kvr):
    """Without kvr_sim_config.extended_policies the lean kernel instantiation runs and an
    extended per-trial policy is refused (status 3) instead of silently misbehaving."""
    import torch
    tr = wl.gsp(4, 4, 0.5, seed=3, W=2)
    dt = kvr.DeviceTrace(tr)
    sim = kvr.Simulator(2, 512)
    pols = kvr.policies_array([kvr.Policy(router=kvr.ROUTE_LBGR_RLS), kvr.Policy(tracker_grain=4),
                               kvr.Policy()])
    b = sim.alloc([dt], 3, 0, dt.device)
    b["keys"].copy_(torch.arange(1, 4, dtype=torch.int64))
    b["policies"].copy_(torch.from_numpy(pols.view(np.uint8)))
    sim.launch([dt], 3, b, with_policies=True)
    out = sim.collect(b, 3)
    assert list(out.results["status"]) == [3, 3, 0]
    assert not sim.cfg.extended_policies


def test_closed_form_routing_p31(kvr, oracle_mod):
    """P31's closed forms through the GPU: cache-aware herding (all on worker 0, hit
    tokens 16 * sum_g (Q-1) p_g) and join-shortest-queue (worker j mod W)."""
    from paper_2601_18999_b200 import workloads as wl
    from parity_util import compare
    G, Q, p, u = 5, 6, (3, 5, 2, 7, 4), 3

    def trace(spacing):
        paths = []
        for k in range(Q):
            for g in range(G):
                paths.append([1000 * (g + 1) + d for d in range(p[g])] +
                             [10 ** 6 + 100 * (k * G + g) + d for d in range(u)])
        return wl.from_paths(paths, arrival_ms=[spacing * j for j in range(len(paths))])

    herd = [kvr.Policy(router=2, tau=1e300, eviction=1), kvr.Policy(router=1, w_load=0.0, w_hit=1.0)]
    out, _ = compare(oracle_mod, kvr, trace(1.0e5), 4, 1000, herd, [3, 4], ring=64)
    for t in range(2):
        assert np.all(out.records[t]["worker"][:G * Q] == 0)
        assert int(out.results[t]["hit_tokens"]) == 16 * sum((Q - 1) * pg for pg in p)
    jsq = [kvr.Policy(router=2, tau=0.0, eviction=0), kvr.Policy(router=1, w_load=1.0, w_hit=0.0)]
    out, _ = compare(oracle_mod, kvr, trace(0.0), 3, 1000, jsq, [5, 6], ring=64)
    for t in range(2):
        assert np.all(out.records[t]["worker"][:G * Q] == np.arange(G * Q) % 3)
