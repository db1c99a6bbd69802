"""Pins of the oracle's continuous-batching engine (beta >= 1; SURVEY §8f #2,
DESIGN.md readings A30-A35) against the paper and textbook queueing facts (no GPU).

P25 hand example (golden/hand_example_p25_batching.txt): pinning, FIFO wait,
    update at dequeue.
P26 FIFO multi-server closed form (Kiefer-Wolfowitz recursion with equal work).
P27 Thm 2 lower-bound construction: L-LRU misses every rotating
    request, OPT one per B-L-beta+2 of them.
P28 reduction: with every query finished before the next arrives, the batched
    engine equals the beta = 1 model of A3/A12 for every beta.
P29 invariants (capacity, pins = in-flight paths, <= beta in flight, conservation)
    under the premise beta * L_max <= B.
"""
import os

import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rr(oracle_mod, **kw):
    return oracle_mod.OraclePolicy(router=oracle_mod.ROUTE_ROUND_ROBIN, **kw)


# -------------------------------------------------------------------------- P25
@pytest.mark.parametrize("eviction", [0, 1])
def test_p25_batching_hand_example(oracle_mod, eviction):
    x, y, z, u, v = 1, 2, 3, 4, 5
    tr = wl.from_paths([[x, y], [x, z], [u, v], [x, y]], arrival_ms=[0.0, 0.5, 1.0, 2.5],
                       block_tokens=1)
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=4, alpha_cached_ms=0.0, alpha_miss_ms=1.0,
                                  out_ms_per_token=0.0, batch_slots=2)
    r = oracle_mod.run(cfg, tr, _rr(oracle_mod, eviction=eviction), 0, record=True,
                       victims_cap=8, check_invariants=True)
    assert r.rc == 0 and r.result["status"] == 0
    rows = [l.split() for l in open(os.path.join(GOLDEN, "hand_example_p25_batching.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 4
    for row in rows:
        j = int(row[0])
        rec = r.records[j]
        assert rec["worker"] == int(row[1]) and rec["hit_tokens"] == int(row[2])
        assert rec["ttft_ms"] == float(row[3]) and rec["latency_ms"] == float(row[4])
        assert rec["n_victims"] == int(row[5])
    ids = oracle_mod.chain(tr)
    assert r.victims[r.records[2]["victim_offset"]] == ids[3]      # z = 2nd block of q1
    res = r.result
    assert res["hit_tokens"] == 3 and res["input_tokens"] == 8 and res["evictions"] == 1
    assert res["makespan_ms"] == 5.0 and res["last_completion_ms"] == 3.5
    assert res["sum_latency_ms"] == 5.5 and res["max_pending"] == 3
    # the beta = 1 model (update at assignment, single server) gives other numbers
    r1 = oracle_mod.run(oracle_mod.OracleConfig(W=1, capacity_blocks=4, alpha_miss_ms=1.0,
                                                out_ms_per_token=0.0),
                        tr, _rr(oracle_mod, eviction=eviction), 0, record=True)
    assert list(r1.records["latency_ms"]) != list(r.records["latency_ms"])


def test_p25b_router_sees_cache_at_arrival(oracle_mod):
    """A32: a query queued but not started has not touched the cache yet, so the
    router's h~ for a later arrival excludes it (STATIC score = -h~/|q|)."""
    a, b, c = 1, 2, 3
    tr = wl.from_paths([[a, b], [a, c], [a, c]], arrival_ms=[0.0, 0.5, 1.0], block_tokens=1)
    pol = oracle_mod.OraclePolicy(router=oracle_mod.ROUTE_STATIC_LINEAR, w_hit=1.0, w_load=0.0)
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=8, alpha_miss_ms=1.0, out_ms_per_token=0.0,
                                  batch_slots=1)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True, check_invariants=True)
    # q1 waits for q0 (done at 2), so at t = 1 the cache is still {a, b}: h~ = 1 of 2
    assert r.records[2]["score"] == -0.5
    # q1 starts at 2 (h = 1, done at 3), q2 starts at 3 and finds a, c: h = 2
    assert list(r.records["hit_tokens"]) == [0, 1, 2]
    assert list(r.records["latency_ms"]) == [2.0, 2.5, 2.0]
    cfg0 = oracle_mod.OracleConfig(W=1, capacity_blocks=8, alpha_miss_ms=1.0, out_ms_per_token=0.0)
    r0 = oracle_mod.run(cfg0, tr, pol, 0, record=True)
    assert r0.records[2]["score"] == -1.0          # A3: updated at assignment


# -------------------------------------------------------------------------- P26
@pytest.mark.parametrize("beta", [1, 2, 3, 5])
def test_p26_fifo_multiserver_closed_form(oracle_mod, beta):
    """All a_j = 0, distinct paths of equal work c (no hits): FIFO over beta
    servers gives latency_k = c * (floor(k / beta) + 1) and TTFT_k =
    latency_k - o|a| (Kiefer-Wolfowitz recursion with equal service)."""
    N, n_in = 11, 2
    paths = [[1000 + 2 * k, 1001 + 2 * k] for k in range(N)]
    tr = wl.from_paths(paths, out_tokens=[3] * N)        # 16-token blocks
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=2 * beta, alpha_miss_ms=1.0,
                                  out_ms_per_token=2.0, batch_slots=beta)
    r = oracle_mod.run(cfg, tr, _rr(oracle_mod, eviction=0), 0, record=True,
                       check_invariants=True)
    assert r.rc == 0 and r.result["status"] == 0
    c = 16.0 * n_in + 2.0 * 3
    for k, rec in enumerate(r.records):
        assert rec["latency_ms"] == c * (k // beta + 1)
        assert rec["ttft_ms"] == c * (k // beta + 1) - 6.0
    assert r.result["last_completion_ms"] == c * ((N - 1) // beta + 1)
    assert r.result["max_pending"] == N
    assert r.result["hit_tokens"] == 0


# -------------------------------------------------------------------------- P27
def _thm2_trace(B, L, beta, cycles, spacing=1.0e5):
    """Thm 2 lower-bound construction: B-L+2 paths with an (L-1)-block
    shared prefix and distinct leaves; batch u = {G_1..G_{beta-1}, G_{u+beta-1}},
    u = 1..B-L-beta+3, looped; a batch arrives at once, after the previous one
    has finished."""
    npaths = B - L + 2
    prefix = [7000 + d for d in range(L - 1)]
    paths, arr, rot = [], [], []
    R = B - L - beta + 3
    t = 0.0
    for _ in range(cycles):
        for u in range(1, R + 1):
            members = list(range(1, beta)) + [u + beta - 1]
            for g in members:
                paths.append(prefix + [9000 + g])
                arr.append(t)
                rot.append(g >= beta)
            t += spacing
    assert max(g for g in range(1, npaths + 1)) == R + beta - 1
    return wl.from_paths(paths, arrival_ms=arr), np.array(rot)


@pytest.mark.parametrize("B,L,beta", [(16, 4, 2), (16, 4, 3), (24, 3, 4)])
def test_p27_thm2_lower_bound_construction(oracle_mod, B, L, beta):
    cycles = 12
    tr, rot = _thm2_trace(B, L, beta, cycles)
    R = B - L - beta + 3                                # rotating paths per cycle
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=B, out_ms_per_token=0.0,
                                  batch_slots=beta, pending_ring=0)
    r = oracle_mod.run(cfg, tr, _rr(oracle_mod, eviction=0), 0, record=True,
                       check_invariants=True)
    assert r.rc == 0 and r.result["status"] == 0
    hit = r.records["hit_tokens"] // 16
    per_batch = beta
    steady = slice(2 * R * per_batch, None)             # after two cycles
    # L-LRU: every rotating request misses exactly its leaf, every fixed one hits
    assert np.all(hit[steady][rot[steady]] == L - 1)
    assert np.all(hit[steady][~rot[steady]] == L)
    lru_steady = int(np.sum(rot[steady]))               # one miss each
    assert lru_steady == (cycles - 2) * R
    # OPT on the same request sequence (Belady, single cache): one miss per
    # R - 1 rotating requests -> ratio -> B - L - beta + 2 (Thm 2 lower bound)
    _, flags = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_OPT)
    per_q = np.add.reduceat(flags, np.arange(0, len(flags), L))
    opt_steady = int(np.sum(per_q[steady]))
    n_rot = lru_steady
    assert abs(opt_steady - n_rot / (R - 1)) <= 2
    assert lru_steady / max(opt_steady, 1) >= (B - L - beta + 2) * (1 - 2.0 * (R - 1) / n_rot) - 1e-9


# -------------------------------------------------------------------------- P28
@pytest.mark.parametrize("router", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("eviction,fallback", [(0, 0), (1, 0), (1, 1), (1, 2)])
def test_p28_spaced_arrivals_reduce_to_beta1_model(oracle_mod, router, eviction, fallback):
    base = wl.gsp(8, 6, 0.5, seed=31 + router)
    tr = wl.from_paths([list(base.block_keys[base.block_offsets[j]:base.block_offsets[j + 1]])
                        for j in range(base.n_queries)],
                       n_out=base.n_out_blocks, out_tokens=base.out_tokens,
                       arrival_ms=[1.0e5 * j for j in range(base.n_queries)])
    pol = oracle_mod.OraclePolicy(eviction=eviction, rlt_fallback=fallback, router=router)
    B = 2 * int(tr.max_blocks) + 3                     # premise 2 L_max <= B holds
    ref = oracle_mod.run(oracle_mod.OracleConfig(W=3, capacity_blocks=B), tr, pol, 5,
                         record=True, victims_cap=4096, check_invariants=True)
    assert ref.rc == 0 and ref.result["evictions"] > 0
    for beta in (1, 2):
        cfg = oracle_mod.OracleConfig(W=3, capacity_blocks=B, batch_slots=beta)
        r = oracle_mod.run(cfg, tr, pol, 5, record=True, victims_cap=3 * 4096,
                           check_invariants=True)
        assert r.rc == 0 and r.result["status"] == 0
        for k in ("queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks",
                  "evictions", "rlt_draws", "rlt_resets", "rlt_fallbacks", "decision_digest"):
            assert r.result[k] == ref.result[k], k
        for k in ("makespan_ms", "last_completion_ms", "max_latency_ms"):
            assert r.result[k] == ref.result[k], k
        for k in ("sum_latency_ms", "sum_ttft_ms", "sum_load_ms"):
            assert r.result[k] == pytest.approx(ref.result[k], rel=1e-12), k
        for f in ("worker", "hit_tokens", "n_victims", "ttft_ms", "latency_ms", "score"):
            assert np.array_equal(r.records[f], ref.records[f]), f
        for j in range(tr.n_queries):
            n = int(ref.records[j]["n_victims"])
            a = ref.victims[ref.records[j]["victim_offset"]:][:n]
            b = r.victims[r.records[j]["victim_offset"]:][:n]
            assert np.array_equal(a, b)


# -------------------------------------------------------------------------- P29
@pytest.mark.parametrize("beta", [1, 2, 4])
@pytest.mark.parametrize("router", [0, 1, 2, 4, 5])
@pytest.mark.parametrize("eviction,fallback", [(0, 0), (1, 0), (1, 1), (1, 2)])
def test_p29_batching_invariants(oracle_mod, beta, router, eviction, fallback):
    tr = wl.random_tree(80, seed=100 + 7 * beta + router, max_len=6, W=2, util=1.5)
    B = beta * int(tr.max_blocks)                      # tightest premise
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=B, batch_slots=beta, pending_ring=0)
    pol = oracle_mod.OraclePolicy(eviction=eviction, rlt_fallback=fallback, router=router)
    r = oracle_mod.run(cfg, tr, pol, 11, record=True, check_invariants=True)
    assert r.rc == 0 and r.result["status"] == 0      # no admission failure under the premise
    res = r.result
    assert res["queries"] == tr.n_queries
    assert res["hit_tokens"] <= res["input_tokens"]
    assert np.all(r.records["ttft_ms"] <= r.records["latency_ms"])
    assert res["inserted_blocks"] - res["evictions"] <= 2 * B   # at most B cached per worker
    assert res["max_pending"] <= 80
    # every query's blocks are either hits or inserts (token accounting)
    assert res["inserted_blocks"] <= int(tr.total_blocks)
    # capacity premise violated -> admission error at validation (rc 2)
    bad = oracle_mod.OracleConfig(W=2, capacity_blocks=B - 1, batch_slots=beta)
    assert oracle_mod.run(bad, tr, pol, 11).rc == 2
