"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Every test names the pin id of DESIGN.md §5 and the
passage it comes from.  None of them re-types the oracle's formula: they use
published known-answer vectors, hand computations, closed forms, textbook
special cases, exact rational arithmetic, brute force and the paper's bounds.
"""
import math
import os
from collections import OrderedDict
from fractions import Fraction

import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------- P1
def test_p1_philox_known_answers(oracle_mod):
    """Random123 Philox4x32-10 KAT vectors (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        assert oracle_mod.philox4x32_10(v[0:4], v[4:6]) == tuple(v[6:10])
        n += 1
    assert n == 3


# --------------------------------------------------------------------------- P2
def _p2_trace():
    A, B, Cc, D, E, X1, X2, X3 = 1, 2, 3, 4, 5, 11, 12, 13
    return wl.from_paths([[A, B, Cc, X1], [A, B, D, X2], [A, B, Cc, E, X3]], n_out=[1, 1, 1],
                         arrival_ms=[0, 0, 30], out_tokens=[4, 4, 4])


@pytest.mark.parametrize("eviction", [0, 1])
def test_p2_hand_example(oracle_mod, eviction):
    """Hand-computed 3-query example (golden/hand_example_p2.txt): Eq. 1, 2, 4-6."""
    tr = _p2_trace()
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=5, out_ms_per_token=2.0)
    pol = oracle_mod.OraclePolicy(eviction=eviction, mu=0.0, rho=1.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True, victims_cap=8, check_invariants=True)
    assert r.rc == 0
    rows = [list(map(float, l.split())) for l in open(os.path.join(GOLDEN, "hand_example_p2.txt"))
            if l.strip() and not l.startswith("#")]
    for row in rows:
        j = int(row[0])
        rec = r.records[j]
        assert rec["worker"] == row[1] and rec["hit_tokens"] == row[2]
        assert rec["ttft_ms"] == row[3] and rec["latency_ms"] == row[4]
        assert rec["score"] == row[5] and rec["n_victims"] == row[6]
    assert r.result["makespan_ms"] == 80.0 and r.result["sum_load_ms"] == 136.0
    assert r.result["hit_tokens"] == 48 and r.result["input_tokens"] == 160
    x1 = oracle_mod.chain(tr)[3]            # identity of X1 (4th block of Gamma_1)
    assert r.victims[0] == x1


# --------------------------------------------------------------------------- P3
def test_p3_eq1_worked_example(oracle_mod):
    """Eq. 1 with App. A constants: |q|=2048, h=1024 -> 1024 ms."""
    p1 = list(range(1, 65))                       # 64 blocks = 1024 tokens
    p2 = p1 + list(range(100, 164))               # 128 blocks = 2048 tokens, first 64 cached
    tr = wl.from_paths([p1, p2], arrival_ms=[0.0, 5000.0])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=256, out_ms_per_token=0.0)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=0), 0, record=True)
    assert r.records[1]["hit_tokens"] == 1024
    assert r.records[1]["ttft_ms"] == 1024.0 and r.records[1]["latency_ms"] == 1024.0


# --------------------------------------------------------------------------- P4
def test_p4_lbgr_score_example(oracle_mod):
    """|q|=2000, h~=(2000,0), P~=(1500,0), theta=0 -> E^=(1500,2000) -> w0.
    P~_0 = 1500 is produced as one decay tick rho=3/4 of the first query's 2000."""
    p = list(range(1, 2001))
    tr = wl.from_paths([p, p], arrival_ms=[0.0, 10.0], block_tokens=1)
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=2048, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=0, rho=0.75, delta_t_ms=10.0, mu=0.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    assert r.records[1]["worker"] == 0 and r.records[1]["score"] == 1500.0
    assert r.records[1]["hit_tokens"] == 2000


# --------------------------------------------------------------------------- P5
@pytest.mark.parametrize("k", list(range(0, 11)))
def test_p5_decay_exact(oracle_mod, k):
    """P~ <- rho P~ every dt (Alg. 2 l.17; rho = 31/32, dt = 20 ms):
    after k ticks P~ = 48 (31/32)^k exactly (exact rationals, k <= 10)."""
    p = [1, 2, 3]
    tr = wl.from_paths([p, p], arrival_ms=[0.0, 20.0 * k + 1.0], out_tokens=[1000, 0])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=8, out_ms_per_token=20.0)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=0.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    exact = Fraction(48) * Fraction(31, 32) ** k
    assert Fraction(r.records[1]["score"]) == exact       # h = |q| -> C^ = 0, theta = 0


# ------------------------------------------------------------------------- P6/P7
def _adv_phase_misses(oracle_mod, B, L, cycles, eviction, key=0, fallback=0):
    from oracle import analysis as an
    tr = wl.adv(B, L, cycles)
    _, flags = oracle_mod.single_replay(tr, B, eviction, fallback, key)
    ph = an.phases(an.flattened_ids(tr), B)
    return an.misses_per_phase(flags, ph)[1:-1]          # steady-state phases


@pytest.mark.parametrize("B,L", [(16, 4), (8, 2), (32, 5)])
def test_p6_thm1_lru_lower_bound_loop(oracle_mod, B, L):
    """Thm 1 construction: L-LRU misses B-L+1 per phase."""
    m = _adv_phase_misses(oracle_mod, B, L, 30, oracle_mod.EVICT_LRU)
    assert len(m) > 5 and np.all(m == B - L + 1)


@pytest.mark.parametrize("B,L", [(16, 4), (8, 2), (32, 5)])
def test_p7_thm1_opt_one_miss_per_phase(oracle_mod, B, L):
    """Thm 1 construction: OPT incurs 1 miss per phase."""
    m = _adv_phase_misses(oracle_mod, B, L, 30, oracle_mod.EVICT_OPT)
    assert len(m) > 5 and np.all(m == 1)


# --------------------------------------------------------------------------- P8
@pytest.mark.slow
def test_p8_rlt_harmonic_on_thm1_loop(oracle_mod):
    """RLT on the Thm 1 loop is classic marking on k+1 = B-L+2 cyclic tails with
    k = B-L+1 slots: expected misses per phase -> H_k (Fiat et al. 1991)."""
    from oracle import analysis as an
    B, L = 16, 4
    allm = []
    for key in range(1, 121):
        allm.extend(_adv_phase_misses(oracle_mod, B, L, 60, oracle_mod.EVICT_RLT, key=key))
    allm = np.array(allm, dtype=np.float64)
    mean, sd = allm.mean(), allm.std(ddof=1)
    Hk = an.harmonic(B - L + 1)
    assert abs(mean - Hk) < 4 * sd / math.sqrt(len(allm)) + 1e-9, (mean, Hk)
    # and within Thm 3's per-phase bound c + c(H_n - H_c) with c = 1, n = B
    assert mean <= 1 + an.harmonic(B) - 1


# --------------------------------------------------------------------------- P9
def test_p9_coupon_collector_opt_gap(oracle_mod):
    """Thm 5 proof: with uniformly random tails, OPT evicts the
    cached tail requested last, so the gap between misses is the time to
    collect the B-L+1 tails cached at the miss out of B-L+2 equally likely ones:
    (B-L+2) H_{B-L+1} = 14 H_13 = 44.52 at B=16, L=4.  The paper prints
    (B-L+2) H_{B-L+2} = 45.52 (off by one coupon; reading A28 in DESIGN.md);
    the measured gap rejects 45.52 and matches 44.52."""
    from oracle import analysis as an
    B, L = 16, 4
    gaps = []
    for seed in range(4):
        tr = wl.adv_rand(B, L, 40000, seed=seed)
        _, flags = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_OPT)
        q_miss = np.nonzero(flags.reshape(-1, L)[:, L - 1])[0]
        q_miss = q_miss[q_miss > 2000]                  # past the cold start
        gaps.extend(np.diff(q_miss).tolist())
    gaps = np.array(gaps, dtype=np.float64)
    expect = (B - L + 2) * an.harmonic(B - L + 1)
    se = gaps.std() / math.sqrt(len(gaps))
    assert abs(gaps.mean() - expect) < 4 * se, (gaps.mean(), expect)


# -------------------------------------------------------------------------- P10
def test_p10_belady_equals_brute_force(oracle_mod):
    """OPT (furthest next use) equals the exhaustive minimum."""
    checked = 0
    for seed in range(150):
        tr = wl.random_tree(7, seed, max_len=3, alphabet=3, max_out=0)
        if tr.total_blocks > 22:
            continue
        for B in (3, 4, 5):
            if tr.max_blocks > B:
                continue
            opt, _ = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_OPT)
            assert opt == oracle_mod.bruteforce_min_misses(tr, B), (seed, B)
            checked += 1
    assert checked > 100


def test_p10b_full_replay_opt_w1(oracle_mod):
    """The full replay with Belady OPT at W = 1 (the offline analysis the GPU runs,
    SURVEY §8f #1): misses equal the exhaustive minimum on tiny traces,
    the single-cache Belady replay on larger ones; W > 1 is refused (P:170 defines
    OPT for one cache)."""
    checked = 0
    for seed in range(120):
        tr = wl.random_tree(7, seed, max_len=3, alphabet=3, max_out=0)
        if tr.total_blocks > 22:
            continue
        for B in (3, 4, 5):
            if tr.max_blocks > B:
                continue
            cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=B)
            r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=oracle_mod.EVICT_OPT), 7)
            assert r.rc == 0
            assert int(r.result["inserted_blocks"]) == oracle_mod.bruteforce_min_misses(tr, B), (seed, B)
            checked += 1
    assert checked > 80
    tr = wl.adv(32, 4, 4, seed=3)
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=32)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=oracle_mod.EVICT_OPT), 1)
    opt, _ = oracle_mod.single_replay(tr, 32, oracle_mod.EVICT_OPT)
    assert r.rc == 0 and int(r.result["inserted_blocks"]) == opt
    cfg2 = oracle_mod.OracleConfig(W=2, capacity_blocks=32)
    assert oracle_mod.run(cfg2, tr, oracle_mod.OraclePolicy(eviction=oracle_mod.EVICT_OPT), 1).rc == 1


# -------------------------------------------------------------------------- P11
@pytest.mark.parametrize("fallback", [0, 1])
def test_p11_rlt_competitive_gate(oracle_mod, fallback):
    """Thm 3 via its proof's per-phase bound c + c(H_n - H_c) and
    Lemma 1's OPT >= max{c/2,1}: E[RLT] <= (2H_B - 1) OPT + B,
    with E[RLT] computed exactly by enumerating every uniform choice."""
    from oracle import analysis as an
    checked = 0
    for seed in range(300):
        tr = wl.random_tree(7, 1000 + seed, max_len=3, alphabet=3, max_out=0)
        if tr.total_blocks > 18:
            continue
        for B in (3, 4):
            if tr.max_blocks > B:
                continue
            mean, var, leaves = oracle_mod.rlt_exact_expectation(tr, B, fallback)
            opt = oracle_mod.bruteforce_min_misses(tr, B)
            assert mean <= (2 * an.harmonic(B) - 1) * opt + B + 1e-9, (seed, B, mean, opt)
            assert mean >= opt - 1e-9                     # no policy beats OPT
            checked += 1
    assert checked > 60


# -------------------------------------------------------------------------- P12
def test_p12_lru_upper_bound(oracle_mod):
    """Thm 1 upper bound: L-LRU <= (B - L + 2) OPT (L = min path length)."""
    for seed in range(200):
        tr = wl.random_tree(12, 2000 + seed, max_len=4, alphabet=3, max_out=1)
        L = int((tr.n_in_blocks + tr.n_out_blocks).min())
        for B in (4, 5, 6):
            if tr.max_blocks > B:
                continue
            lru, _ = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_LRU)
            opt, _ = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_OPT)
            assert lru <= (B - L + 2) * opt, (seed, B, lru, opt)
            assert opt <= lru


# -------------------------------------------------------------------------- P13
@pytest.mark.parametrize("eviction,fallback", [(0, 0), (1, 0), (1, 1), (1, 2)])
@pytest.mark.parametrize("router", [0, 1, 2, 3, 4])
def test_p13_invariants(oracle_mod, eviction, fallback, router):
    """Capacity, prefix closure, T subset S, Eq. 3 (others unchanged), hit <= |q|,
    hits+inserted = |Gamma|, P~ >= 0, TTFT <= latency (checked in-oracle every
    query) and makespan >= sum_i P_i / W."""
    for seed in range(6):
        tr = wl.random_tree(120, 3000 + seed, max_len=7, alphabet=3, max_out=2, W=3)
        cfg = oracle_mod.OracleConfig(W=3, capacity_blocks=9, out_ms_per_token=2.0)
        pol = oracle_mod.OraclePolicy(eviction=eviction, rlt_fallback=fallback, router=router)
        r = oracle_mod.run(cfg, tr, pol, seed + 1, check_invariants=True)
        assert r.rc == 0 and r.result["status"] == 0
        res = r.result
        assert res["makespan_ms"] >= res["sum_load_ms"] / 3 - 1e-9
        assert res["hit_tokens"] <= res["input_tokens"]
        assert res["queries"] == tr.n_queries


# -------------------------------------------------------------------------- P14
def test_p14_all_zero_arrivals_latency_decomposition(oracle_mod):
    """All a_j = 0: E_ij = Cost_ij + P_i^(j-1) bit for bit, TTFT = P + pre."""
    tr = wl.gsp(10, 6, 0.5, seed=5, rate_per_s=0.0)
    cfg = oracle_mod.OracleConfig(W=3, capacity_blocks=300, out_ms_per_token=20.0, pending_ring=0)
    for ev in (0, 1):
        r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=ev), 7, record=True)
        P = [0.0, 0.0, 0.0]
        for j, rec in enumerate(r.records):
            q = 16 * int(tr.n_in_blocks[j])
            pre = 1.0 * float(q - int(rec["hit_tokens"]))
            cost = pre + 20.0 * float(tr.out_tokens[j])
            i = int(rec["worker"])
            assert rec["latency_ms"] == P[i] + cost
            assert rec["ttft_ms"] == P[i] + pre
            P[i] = P[i] + cost
        assert r.result["makespan_ms"] == max(P)


# -------------------------------------------------------------------------- P15
def test_p15_graham_list_scheduling(oracle_mod):
    """alpha_C = alpha_M, o = 0, a = 0, theta = 0, mu = 0, rho = 1: LBGR is Graham's
    list scheduling (argmin load, lowest index on ties); makespan within
    [max(sum/W, max cost), (2 - 1/W) OPT]."""
    W = 4
    tr = wl.gsp(17, 5, 0.5, seed=11, rate_per_s=0.0)
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=300, alpha_cached_ms=1.0, alpha_miss_ms=1.0,
                                  out_ms_per_token=0.0, pending_ring=0)
    pol = oracle_mod.OraclePolicy(eviction=1, est_alpha_cached_ms=1.0, est_alpha_miss_ms=1.0,
                                  mu=0.0, rho=1.0)
    r = oracle_mod.run(cfg, tr, pol, 3, record=True)
    loads = [0] * W
    for j, rec in enumerate(r.records):
        c = 16 * int(tr.n_in_blocks[j])
        i = min(range(W), key=lambda k: (loads[k], k))
        assert rec["worker"] == i
        loads[i] += c
    costs = 16 * tr.n_in_blocks.astype(np.int64)
    lb = max(costs.sum() / W, costs.max())
    assert r.result["makespan_ms"] == max(loads)
    # Graham (1966): makespan <= sum/W + (1 - 1/W) max <= (2 - 1/W) OPT
    assert lb <= r.result["makespan_ms"] <= costs.sum() / W + (1 - 1 / W) * costs.max()


# -------------------------------------------------------------------------- P16
def test_p16_flat_cache_is_textbook_lru(oracle_mod):
    """W = 1, one block per query: the tree is flat and L-LRU is textbook LRU
    paging; RLT is classic marking whose U is never empty."""
    rng = np.random.default_rng(0)
    for B in (3, 5, 8):
        pages = rng.integers(0, B + 3, size=400).tolist()
        tr = wl.from_paths([[p] for p in pages])
        lru, flags = oracle_mod.single_replay(tr, B, oracle_mod.EVICT_LRU)
        od, misses, ref = OrderedDict(), 0, []
        for p in pages:
            if p in od:
                od.move_to_end(p)
                ref.append(0)
            else:
                misses += 1
                ref.append(1)
                if len(od) == B:
                    od.popitem(last=False)
                od[p] = True
        assert lru == misses and flags.tolist() == ref
        # cyclic B+1 pages: LRU misses every access
        cyc = wl.from_paths([[k % (B + 1)] for k in range(10 * (B + 1))])
        assert oracle_mod.single_replay(cyc, B, oracle_mod.EVICT_LRU)[0] == 10 * (B + 1)
        cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=B)
        r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=1, router=3), 5)
        assert r.result["rlt_fallbacks"] == 0 and r.result["inserted_blocks"] >= lru * 0


# -------------------------------------------------------------------------- P17
def test_p17_round_robin_counts(oracle_mod):
    tr = wl.gsp(7, 9, 0.5, seed=2)
    for W in (1, 3, 4, 5):
        cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=300)
        r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(router=3), 1, record=True)
        counts = np.bincount(r.records["worker"], minlength=W)
        N = tr.n_queries
        assert set(counts.tolist()) <= {N // W, -(-N // W)}
        assert np.all(r.records["worker"] == np.arange(N) % W)


# -------------------------------------------------------------------------- P18
@pytest.mark.parametrize("mu", [0.3, 0.992, 1.7])
def test_p18_online_update_reduces_residual(oracle_mod, mu):
    """OnlineUpdate minimises (E - E^)^2: one step with 0 < mu < 2 on a
    sample strictly shrinks that sample's residual; a zero residual leaves theta
    unchanged (same features -> same score)."""
    p1, p2, p3 = [1, 2, 3, 4], [5, 6, 7, 8], [9, 10, 11, 12]
    tr = wl.from_paths([p1, p2, p3], arrival_ms=[0.0, 1000.0, 2000.0], out_tokens=[3, 3, 3])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=16, out_ms_per_token=5.0)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=mu, rho=1.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    rec = r.records
    E = rec["latency_ms"]
    assert E[0] == E[1] == E[2]                          # identical service, empty queue
    r0, r1 = E[0] - rec["score"][0], E[1] - rec["score"][1]
    assert r0 != 0 and abs(r1) < abs(r0)
    # zero residual: with the estimator equal to the truth the score never moves
    cfg0 = oracle_mod.OracleConfig(W=1, capacity_blocks=16, out_ms_per_token=0.0)
    r0run = oracle_mod.run(cfg0, tr, pol, 0, record=True)
    assert np.all(r0run.records["score"] == r0run.records["latency_ms"])


# -------------------------------------------------------------------------- P19
def test_p19_table2_direction(oracle_mod):
    """Table 2, directional only: one worker, worst-case round-robin
    GSP order, working set >> B: RLT hit rate >= 2x L-LRU hit rate."""
    tr = wl.gsp(24, 16, 0.5, seed=4, order="rr", lengths=(256, 512, 1024))
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=256, pending_ring=0)
    hits = {}
    for ev in (0, 1):
        tot = 0
        for key in range(4):
            r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=ev, router=3), key + 1)
            tot += r.result["hit_tokens"]
        hits[ev] = tot
    assert hits[1] >= 2 * hits[0], hits


# -------------------------------------------------------------------------- P20
def test_p20_determinism(oracle_mod):
    tr = wl.gsp(10, 10, 0.5, seed=9)
    cfg = oracle_mod.OracleConfig(W=4, capacity_blocks=300)
    a = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(), 42, record=True)
    b = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(), 42, record=True)
    assert a.result == b.result and a.records.tobytes() == b.records.tobytes()
    c = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(), 43)
    assert c.result["decision_digest"] != a.result["decision_digest"]


# -------------------------------------------------------------------------- P21
def test_p21_block_identity_contract_kat(oracle_mod):
    """Known-answer vectors of the block-identity contract (golden/identity_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "identity_kat.txt"))
            if l.strip() and not l.startswith("#")]
    for row in rows:
        if row[0] == "fmix64":
            assert oracle_mod.fmix64(int(row[1], 16)) == int(row[2], 16)
        else:
            keys = [int(x) for x in row[1].split(",")]
            tr = wl.from_paths([keys])
            assert [int(h) for h in oracle_mod.chain(tr)] == [int(x, 16) for x in row[2:]]
    # fmix64 is a bijection (MurmurHash3 finalizer): no collisions on 2^16 inputs
    xs = [oracle_mod.fmix64(k) for k in range(1 << 12)]
    assert len(set(xs)) == len(xs)


def test_p21_prefix_property(oracle_mod):
    """Identities encode the whole prefix: equal prefixes -> equal
    identities, one differing block changes every later identity."""
    tr = wl.from_paths([[1, 2, 3, 4], [1, 2, 9, 4], [1, 2, 3, 4]])
    h = oracle_mod.chain(tr).reshape(3, 4)
    assert np.all(h[0] == h[2]) and np.all(h[0, :2] == h[1, :2])
    assert np.all(h[0, 2:] != h[1, 2:])


# -------------------------------------------------------------------------- P22
@pytest.mark.parametrize("key,victim_block", [(0, 1), (2, 2), (12, 3)])
def test_p22_rlt_draw_slot_order_kat(oracle_mod, key, victim_block):
    """RLT draw contract: after the reset at the 5th mark (Alg. 1 l.8-9), U is
    {AB, C, D} in slot order; Philox(K,(0,0,1)) picks index floor(r*3/2^64)."""
    tr = wl.from_paths([[1, 2], [3], [4], [5]])
    H = oracle_mod.chain(tr)               # A, AB, C, D, E
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=4)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=1, router=3), key,
                       record=True, victims_cap=4)
    assert r.result["rlt_resets"] == 1 and r.result["rlt_draws"] == 1
    assert r.victims[0] == H[victim_block]
    r64 = oracle_mod.philox4x32_10([0, 0, 0, 1], [key & 0xFFFFFFFF, key >> 32])
    r64 = r64[0] | (r64[1] << 32)
    assert (r64 * 3) >> 64 == victim_block - 1


# -------------------------------------------------------------------------- P23
@pytest.mark.parametrize("lam", [1.0, 0.992, 0.97])   # (1/lam)^n bounds rounding growth
def test_p23_rls_step_is_weighted_least_squares(oracle_mod, lam):
    """The LBGR_RLS residual model (reading A8b of "learning rate 0.992"; the
    squared-loss objective of P:361): n sequential RLS steps from P0 = p0*I,
    theta0 = 0 equal the closed-form exponentially weighted least squares
    argmin sum_t lam^(n-t) (y_t - phi_t' theta)^2 + lam^n/p0 |theta|^2."""
    rng = np.random.default_rng(23)
    n, p0 = 200, 1e6
    X = np.column_stack([rng.normal(size=(n, 3)), np.ones(n)])
    y = X @ np.array([0.5, -2.0, 1.25, 3.0]) + 0.1 * rng.normal(size=n)
    P = np.eye(4) * p0
    th = np.zeros(4)
    for t in range(n):
        oracle_mod.rls_step(P, th, X[t], y[t] - X[t] @ th, lam)
    w = lam ** (n - 1 - np.arange(n))
    A = (X * w[:, None]).T @ X + (lam ** n / p0) * np.eye(4)
    ref = np.linalg.solve(A, (X * w[:, None]).T @ y)
    assert np.allclose(th, ref, rtol=1e-7, atol=1e-9), (th, ref)
    # P starts at 1e6*I: the first steps cancel ~6 digits, later ones amplify by 1/lam
    assert np.allclose(P, np.linalg.inv(A), rtol=1e-4, atol=1e-10)


# -------------------------------------------------------------------------- P24
def _record_run(oracle_mod, tr, W, B, pol, key=5):
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=B)
    r = oracle_mod.run(cfg, tr, pol, key, record=True)
    assert r.rc == 0
    return r


def test_p24_tracker_lag_hand_example(oracle_mod):
    """App. E: the global tracker can be stale.  Reading A29 with
    tracker_lag = 1: the router has not yet seen the previous query's update.
    Two workers, STATIC router (w_load = w_hit = 1), the same 3-block path twice
    (both arrive at t = 0, so query 0 is still pending at query 1):
      live view:  worker 0 scores 1*1 - 1*1 = 0, worker 1 scores 0 -> tie -> worker 0, full hit;
      lagged:     worker 0 scores 1*1 - 0   = 1, worker 1 scores 0 -> worker 1, no hit."""
    tr = wl.from_paths([[11, 12, 13], [11, 12, 13]])
    base = dict(router=oracle_mod.ROUTE_STATIC_LINEAR, w_hit=1.0, w_load=1.0, eviction=0)
    live = _record_run(oracle_mod, tr, 2, 8, oracle_mod.OraclePolicy(**base))
    lag = _record_run(oracle_mod, tr, 2, 8, oracle_mod.OraclePolicy(tracker_lag=1, **base))
    assert list(live.records["worker"]) == [0, 0] and list(lag.records["worker"]) == [0, 1]
    assert list(live.records["hit_tokens"]) == [0, 3 * 16] and list(lag.records["hit_tokens"]) == [0, 0]


def test_p24_tracker_grain_reduces_to_no_hit_term(oracle_mod):
    """A29 grain larger than every path: the tracker sees no hits, so STATIC with
    w_hit = 1 routes exactly like STATIC with w_hit = 0 and an exact tracker;
    grain = 1, lag = 0 is the default replay bit for bit."""
    tr = wl.gsp(12, 8, 0.5, seed=0x24, W=4)
    big = max(int(tr.n_in_blocks.max()) + 1, 2)
    a = _record_run(oracle_mod, tr, 4, 512, oracle_mod.OraclePolicy(
        router=oracle_mod.ROUTE_STATIC_LINEAR, w_hit=1.0, tracker_grain=big))
    b = _record_run(oracle_mod, tr, 4, 512, oracle_mod.OraclePolicy(
        router=oracle_mod.ROUTE_STATIC_LINEAR, w_hit=0.0))
    assert np.array_equal(a.records["worker"], b.records["worker"])
    assert a.result["decision_digest"] == b.result["decision_digest"]
    c = _record_run(oracle_mod, tr, 4, 512, oracle_mod.OraclePolicy(tracker_grain=1, tracker_lag=0))
    d = _record_run(oracle_mod, tr, 4, 512, oracle_mod.OraclePolicy())
    assert c.result["decision_digest"] == d.result["decision_digest"]


# -------------------------------------------------------------------------- P30
def test_p30_collision_check(oracle_mod):
    """Identity collision check: a crafted genuine 64-bit collision of
    two different depth-2 prefixes (tests/collision_util.py) is found -- the chain
    really gives both the same identity -- and normal traces report none."""
    from collision_util import colliding_pair, fmix64, fmix64_inv
    for x in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
        assert fmix64_inv(fmix64(x)) == x and oracle_mod.fmix64(x) == fmix64(x)
    a1, a2, b1 = 11, 12, 13
    b2 = colliding_pair(a1, a2, b1)
    tr = wl.from_paths([[a1, a2], [b1, b2], [a1, a2, 5]], n_out=[0, 0, 1])
    H = oracle_mod.chain(tr)
    assert H[1] == H[3] and H[0] != H[2]              # one identity, two prefixes
    # occurrences of that identity, in CSR order: [a1,a2]@1, [b1,b2]@3, [a1,a2,..]@5
    # -> adjacent pairs (1,3) and (3,5) differ in parent/key: 2 collisions
    assert oracle_mod.count_collisions(tr) == 2
    tr.hash_salt = 77                                  # re-salting dissolves it
    assert oracle_mod.count_collisions(tr) == 0
    for t in (wl.gsp(20, 10, 0.5, seed=1), wl.mt(12, 0.5, seed=2), wl.random_tree(300, 3)):
        assert oracle_mod.count_collisions(t) == 0


# -------------------------------------------------------------------------- P31
def _groups_trace(G=5, Q=6, p=(3, 5, 2, 7, 4), u=3, spacing=1.0e5):
    """G groups, group g's queries share a p[g]-block prefix then u unique blocks;
    queries interleaved g = 0..G-1 round after round."""
    paths = []
    for k in range(Q):
        for g in range(G):
            paths.append([1000 * (g + 1) + d for d in range(p[g])] +
                         [10 ** 6 + 100 * (k * G + g) + d for d in range(u)])
    return wl.from_paths(paths, arrival_ms=[spacing * j for j in range(len(paths))]), p, G, Q


@pytest.mark.parametrize("router,kw", [(2, dict(tau=1e300)), (1, dict(w_load=0.0, w_hit=1.0))])
def test_p31_cache_aware_herding(oracle_mod, router, kw):
    """Pure cache affinity (THRESHOLD that never balances, STATIC without a load term)
    is greedy argmax-h with lowest-index ties: every query lands on worker 0, which
    then holds every group's prefix -> hit tokens = 16 * sum_g (Q-1) p_g (no
    evictions at ample B).  The heuristics of P:41 at their hit-rate extreme."""
    tr, p, G, Q = _groups_trace()
    cfg = oracle_mod.OracleConfig(W=4, capacity_blocks=1000, pending_ring=0)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(router=router, eviction=1, **kw), 3,
                       record=True, check_invariants=True)
    assert np.all(r.records["worker"] == 0)
    assert r.result["hit_tokens"] == 16 * sum((Q - 1) * pg for pg in p)
    assert r.result["evictions"] == 0
    assert r.result["sum_load_ms"] == r.result["makespan_ms"]     # one loaded worker


@pytest.mark.parametrize("router,kw", [(2, dict(tau=0.0)), (1, dict(w_load=1.0, w_hit=0.0))])
@pytest.mark.parametrize("W", [2, 3, 5])
def test_p31_join_shortest_queue(oracle_mod, router, kw, W):
    """All a_j = 0, so nothing completes: pure load balancing on pending counts
    (THRESHOLD with tau = 0, STATIC without a hit term) is join-the-shortest-queue
    with lowest-index ties, i.e. worker j mod W."""
    tr, _, _, _ = _groups_trace(spacing=0.0)
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=1000, pending_ring=0)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(router=router, eviction=0, **kw), 3,
                       record=True, check_invariants=True)
    assert np.all(r.records["worker"] == np.arange(tr.n_queries) % W)


# -------------------------------------------------------------------------- P32
def _constant_feature_trace(n=40, L=4, gap=1.0e5):
    """Unique equal-length paths, spaced so every query finishes (and releases its load,
    rho = 1) before the next arrives: phi = (0, 16L/1000, 0, 1) and E = cost every time."""
    paths = [[100 * j + d for d in range(L)] for j in range(n)]
    return wl.from_paths(paths, arrival_ms=[gap * j for j in range(n)], out_tokens=[3] * n)


@pytest.mark.parametrize("mu", [0.05, 0.5, 0.992, 1.5])
def test_p32_nlms_trajectory_closed_form(oracle_mod, mu):
    """NLMS (A8) with constant features phi and constant target E: the residual
    r_j = E - E^_j obeys r_{j+1} = r_j (1 - mu |phi|^2 / (1 + |phi|^2)) exactly in real
    arithmetic (theta moves along phi only) -> geometric decay, checked over 40 steps."""
    tr = _constant_feature_trace()
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=64, out_ms_per_token=5.0)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=0, mu=mu, rho=1.0), 0, record=True)
    E, Eh = r.records["latency_ms"], r.records["score"]
    assert np.all(E == E[0])
    phi = np.array([0.0, 16 * 4 / 1000.0, 0.0, 1.0])
    g = 1.0 - mu * (phi @ phi) / (1.0 + phi @ phi)
    res = E - Eh
    pred = res[0] * g ** np.arange(len(res))
    assert np.allclose(res, pred, rtol=1e-9, atol=1e-9 * abs(res[0]))


@pytest.mark.parametrize("lam,p0", [(0.992, 1000.0), (0.5, 10.0), (1.0, 1.0)])
def test_p32_rls_trajectory_closed_form(oracle_mod, lam, p0):
    """RLS (A8b) with constant phi: s_j = phi' P_j phi follows s_{j+1} = s_j / (lam + s_j)
    from s_0 = p0 |phi|^2 and the residual r_{j+1} = r_j lam / (lam + s_j)."""
    tr = _constant_feature_trace()
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=64, out_ms_per_token=5.0)
    pol = oracle_mod.OraclePolicy(eviction=0, router=oracle_mod.ROUTE_LBGR_RLS, mu=lam,
                                  rls_p0=p0, rho=1.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    res = r.records["latency_ms"] - r.records["score"]
    phi = np.array([0.0, 16 * 4 / 1000.0, 0.0, 1.0])
    s = p0 * (phi @ phi)
    pred = [res[0]]
    for _ in range(len(res) - 1):
        pred.append(pred[-1] * lam / (lam + s))
        s = s / (lam + s)
    pred = np.array(pred)
    scale = abs(res[0])
    assert np.allclose(res, pred, rtol=1e-8, atol=1e-8 * scale)
