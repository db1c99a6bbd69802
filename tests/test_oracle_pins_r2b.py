"""Pins of the oracle functions added in round 2 for the SURVEY §8(f) rows.

P38  the SGLang-style cache-aware router ("switches between the
     highest-hit-rate and the least-loaded routing based on a predefined heuristic
     load-balance threshold"; reading A38): each of its three branches reduced to a
     closed-form routing sequence.
P39  the k-event stale tracker (App. E P:1229 "staleness ... caused by concurrent
     updates"; reading A29 with k >= 1): an anti-affinity router whose decisions
     reveal exactly which past cache state the router sees, for k = 1..6.
P40  the phase ledger (reading A39): a hand example, the Thm 1 loop
     (clean = 1 and B-L+1 misses per L-LRU phase, 1 per OPT phase), the
     phase partition against an independent Python split, Lemma 2 / Lemma 3 on random
     trees, and Lemma 1 in its summed form (A23) against Belady OPT.

Every expected value is derived in the docstring or is a closed form / a lemma of the
paper; none comes from running the oracle.
"""
import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl


def _spaced(paths, gap=1e6):
    """Queries far apart in time: every query completes before the next arrives."""
    return wl.from_paths(paths, arrival_ms=[gap * j for j in range(len(paths))])


def _workers(oracle_mod, tr, W, B, **pol):
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=B)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=0, **pol), 1, record=True)
    assert r.rc == 0
    return [int(x) for x in r.records["worker"]]


# --------------------------------------------------------------------------- P38
CA = dict(router=6)


def test_p38_imbalance_branch_is_join_shortest_queue(oracle_mod):
    """abs = -1, rel = 0: the load counts as imbalanced as soon as any query is pending
    (max - min > -1 and max > 0).  All arrivals at t = 0 and nothing completes, so from
    the second query on the rule is join-the-shortest-queue with lowest-index ties:
    i*_j = j mod W.  The first query sees no load (max = 0), takes the cache branch with
    no match (rate 0 <= 0.5) and then the fewest cached blocks: all 0 -> worker 0."""
    W = 3
    paths = [[100 * j + d for d in range(4)] for j in range(10)]
    tr = wl.from_paths(paths, arrival_ms=[0.0] * 10)
    got = _workers(oracle_mod, tr, W, 64, ca_balance_abs=-1.0, ca_balance_rel=0.0, **CA)
    assert got == [j % W for j in range(10)]


def test_p38_cache_branch_herds_on_highest_match(oracle_mod):
    """abs huge (never imbalanced), threshold -1 (every match rate exceeds it): the
    highest match wins, ties to the lowest index.  Query 0 matches nothing anywhere ->
    worker 0; every later query shares block 0 with all earlier ones, so worker 0 keeps
    the highest match: all queries on worker 0 (the pure cache-affinity closed form of
    P31)."""
    paths = [[7] + [100 * j + d for d in range(1, 4)] for j in range(8)]
    got = _workers(oracle_mod, _spaced(paths), 4, 64, ca_balance_abs=1e18,
                   ca_cache_threshold=-1.0, **CA)
    assert got == [0] * 8


def test_p38_fewest_cached_blocks_branch(oracle_mod):
    """abs huge, threshold 2 (a rate <= 1 never exceeds it): always the worker with the
    fewest cached blocks.  Unique 4-block paths, B = 16: workers fill round-robin
    (sizes 0,0,0 -> w0; 4,0,0 -> w1; ...), 4 queries each fill a cache; after 12 queries
    every cache holds 16 blocks and the lowest index wins forever."""
    W, B, n = 3, 16, 4
    paths = [[1000 * j + d for d in range(n)] for j in range(20)]
    got = _workers(oracle_mod, _spaced(paths), W, B, ca_balance_abs=1e18,
                   ca_cache_threshold=2.0, **CA)
    fill = W * B // n
    assert got == [j % W for j in range(fill)] + [0] * (20 - fill)


def test_p38_threshold_is_strict(oracle_mod):
    """W = 2, B = 64, balanced.  q0 = [1,2,3,4] -> w0 (nothing cached, fewest blocks:
    tie -> w0).  q1 = [1,2,5,6]: highest match w0 with h = 2 blocks of 4 = rate 0.5.
    Threshold 0.5 (strict >): not above -> fewest cached blocks: w1 (0 < 4).  Threshold
    0.49: above -> w0."""
    tr = _spaced([[1, 2, 3, 4], [1, 2, 5, 6]])
    assert _workers(oracle_mod, tr, 2, 64, ca_balance_abs=1e18, ca_cache_threshold=0.5, **CA) == [0, 1]
    assert _workers(oracle_mod, tr, 2, 64, ca_balance_abs=1e18, ca_cache_threshold=0.49, **CA) == [0, 0]


def test_p38_balance_needs_both_thresholds(oracle_mod):
    """Arrivals at 0 (nothing completes: load = queries assigned so far), threshold 2
    (the balanced branch always takes the fewest cached blocks), W = 2, paths of
    4, 4, 12, 4, 4, 4 unique blocks.  L = pending loads, S = cached blocks.
    abs = 1.5, rel = 1 (a difference of 1 is never imbalanced):
      q0 (0,0) -> S tie -> w0; q1 S (4,0) -> w1; q2 S (4,4) tie -> w0; q3 S (16,4) -> w1;
      q4 S (16,8) -> w1; q5 L (2,3) diff 1 -> S (16,12) -> w1:  0 1 0 1 1 1.
    abs = 0.5, rel = 1 (imbalanced iff the loads differ):
      q1 L (1,0) -> least loaded w1; q2 L (1,1) -> S (4,4) tie -> w0; q3 L (2,1) -> w1;
      q4 L (2,2) -> S (16,8) -> w1; q5 L (2,3) -> least loaded w0:  0 1 0 1 1 0.
    abs = 0.5, rel = 2 (also needs max > 2 min): q1 L (1,0): 1 > 0 -> w1; q3 L (2,1):
      2 > 2 false -> S (16,4) -> w1; q5 L (2,3): 3 > 4 false -> S (16,12) -> w1:
      0 1 0 1 1 1 -- the relative threshold alone blocks the switch at q5."""
    lens = [4, 4, 12, 4, 4, 4]
    paths = [[100 * j + d for d in range(n)] for j, n in enumerate(lens)]
    tr = wl.from_paths(paths, arrival_ms=[0.0] * len(lens))
    run = lambda a, r: _workers(oracle_mod, tr, 2, 64, ca_cache_threshold=2.0,  # noqa: E731
                                ca_balance_abs=a, ca_balance_rel=r, **CA)
    assert run(1.5, 1.0) == [0, 1, 0, 1, 1, 1]
    assert run(0.5, 1.0) == [0, 1, 0, 1, 1, 0]
    assert run(0.5, 2.0) == [0, 1, 0, 1, 1, 1]


# --------------------------------------------------------------------------- P39
ANTI = dict(router=1, w_load=0.0, w_hit=-1.0)   # STATIC with a negative hit weight: s = +h~/|q|


@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_p39_stale_tracker_identical_queries(oracle_mod, k):
    """Anti-affinity (the router prefers the worker it believes holds LESS of the query)
    on one path repeated, spaced.  At query j the router sees the caches after query
    j-1-k.  q0 -> w0 (tie).  For j <= k the update of q0 is unseen -> tie -> w0.  For
    k+1 <= j <= 2k+1 it sees w0 holding the path but not w1's first update (made at
    q_{k+1}) -> w1.  From j = 2k+2 both hold it -> tie -> w0."""
    n = 4 * k + 6
    tr = _spaced([[5, 6, 7, 8]] * n)
    got = _workers(oracle_mod, tr, 2, 64, tracker_lag=k, **ANTI)
    assert got == [0] * (k + 1) + [1] * (k + 1) + [0] * (n - 2 * k - 2)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_p39_stale_tracker_sees_exactly_k_back(oracle_mod, k):
    """k+1 unique paths X_0..X_k all go to w0 (nothing matches anywhere, tie).  A probe
    at j = k+1 is answered from the caches after query j-1-k = 0:
      probe X_0: w0 already holds X_0 -> w1 (a lag of k+1 would see empty caches -> w0);
      probe X_1: w0 does not yet hold X_1 -> tie -> w0 (a lag of k-1 would see it -> w1)."""
    X = [[1000 * i + d for d in range(3)] for i in range(k + 1)]
    assert _workers(oracle_mod, _spaced(X + [X[0]]), 2, 64, tracker_lag=k, **ANTI)[-1] == 1
    assert _workers(oracle_mod, _spaced(X + [X[1]]), 2, 64, tracker_lag=k, **ANTI)[-1] == 0
    # k = 0 (no lag) sees everything: both probes are cached on w0 -> w1
    assert _workers(oracle_mod, _spaced(X + [X[1]]), 2, 64, tracker_lag=0, **ANTI)[-1] == 1


def test_p39_lag_beyond_max_is_refused(oracle_mod):
    tr = _spaced([[1, 2]])
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=8)
    assert oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(tracker_lag=oracle_mod.MAX_TRACKER_LAG), 1).rc == 0
    assert oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(tracker_lag=oracle_mod.MAX_TRACKER_LAG + 1), 1).rc == 1


# --------------------------------------------------------------------------- P40
def test_p40_hand_example(oracle_mod):
    """B = 3, one-block paths a b c d a b (W = 1, Leaf-LRU = textbook LRU, P16).
    Phases {a b c} | {d a b}.  Phase 1: 3 distinct, 3 misses, all first appearances, all
    clean (empty cache).  Phase 2: the cache at its start is {a, b, c}; d is clean and
    evicts a (LRU), a misses and evicts b, b misses: 3 misses at first appearances, but
    only d is clean (a and b were cached when the phase began)."""
    tr = wl.from_paths([[1], [2], [3], [4], [1], [2]], arrival_ms=[0.0] * 6)
    led = oracle_mod.phase_ledger(tr, 3, oracle_mod.EVICT_LRU)
    assert led.tolist() == [[3, 3, 3, 3], [3, 3, 3, 1]]


@pytest.mark.parametrize("B,L", [(16, 4), (8, 2), (32, 5)])
def test_p40_thm1_loop(oracle_mod, B, L):
    """Thm 1 construction: B-L+2 paths = a shared (L-1)-block prefix + a
    distinct tail, cyclic.  A phase holds the prefix and B-L+1 tails.  L-LRU keeps the
    B-L+1 most recent tails, i.e. exactly the ones the next phase does not start with:
    per steady phase c = 1 clean tail, B-L+1 misses, all at first appearances (Lemma 3:
    no old token misses), so Lemma 2's B-L+c is tight.  OPT misses once per phase (P7)."""
    tr = wl.adv(B, L, 12)
    lru = oracle_mod.phase_ledger(tr, B, oracle_mod.EVICT_LRU)[1:-1]
    assert len(lru) > 5
    assert np.all(lru[:, 0] == B) and np.all(lru[:, 3] == 1)
    assert np.all(lru[:, 1] == B - L + 1) and np.all(lru[:, 2] == lru[:, 1])
    opt = oracle_mod.phase_ledger(tr, B, oracle_mod.EVICT_OPT)[1:-1]
    assert np.all(opt[:, 1] == 1)


def _random_tree_trace(seed, n_paths, max_len, fanout):
    rng = np.random.default_rng(seed)
    paths = []
    for _ in range(n_paths):
        L = int(rng.integers(2, max_len + 1))
        paths.append([int(rng.integers(0, fanout)) + 10 * d for d in range(L)])
    return wl.from_paths(paths, arrival_ms=[0.0] * n_paths)


@pytest.mark.parametrize("seed", range(6))
def test_p40_partition_and_counts(oracle_mod, seed):
    """The ledger's phases equal an independent Python greedy split (oracle/analysis.py:
    B distinct ids per phase); the per-phase misses sum to single_replay's total and to
    its per-access flags; 0 <= clean <= first_misses <= distinct, first_misses <= misses."""
    from oracle import analysis as an
    tr = _random_tree_trace(seed, 60, 6, 3)
    B = 8
    ids = an.flattened_ids(tr)
    ph = an.phases(ids, B)
    for ev in (oracle_mod.EVICT_LRU, oracle_mod.EVICT_RLT, oracle_mod.EVICT_OPT):
        led = oracle_mod.phase_ledger(tr, B, ev, philox_key=seed)
        assert len(led) == len(ph)
        assert [int(x) for x in led[:, 0]] == [len(set(ids[a:b].tolist())) for a, b in ph]
        total, flags = oracle_mod.single_replay(tr, B, ev, philox_key=seed)
        assert int(led[:, 1].sum()) == total
        assert [int(x) for x in led[:, 1]] == [int(flags[a:b].sum()) for a, b in ph]
        assert np.all(led[:, 3] <= led[:, 2]) and np.all(led[:, 2] <= led[:, 0])
        assert np.all(led[:, 2] <= led[:, 1])


@pytest.mark.parametrize("seed", range(8))
def test_p40_lemmas_2_3_on_random_trees(oracle_mod, seed):
    """Single-query L-LRU on random prefix trees: Lemma 3, no old token is a
    miss (misses == first_misses) and Lemma 2, misses <= B - L + c in every phase v >= 2,
    L the minimum path length."""
    tr = _random_tree_trace(100 + seed, 80, 7, 3)
    B = 10
    L = int(min(tr.n_in_blocks + tr.n_out_blocks))
    led = oracle_mod.phase_ledger(tr, B, oracle_mod.EVICT_LRU)
    assert np.all(led[:, 1] == led[:, 2])
    assert np.all(led[1:, 1].astype(int) <= B - L + led[1:, 3].astype(int))


@pytest.mark.parametrize("seed", range(8))
def test_p40_lemma1_summed_against_opt(oracle_mod, seed):
    """Lemma 1 in its summed form (A23): over the phases v >= 2, OPT's
    misses >= sum_v max(c_v/2, 1) - 1, with c_v the clean count of L-LRU's phases
    (the same partition; OPT's misses counted over the whole sequence from phase 2 on;
    the -1 absorbs the amortisation across the first boundary)."""
    tr = _random_tree_trace(200 + seed, 80, 6, 3)
    B = 8
    lru = oracle_mod.phase_ledger(tr, B, oracle_mod.EVICT_LRU)
    opt = oracle_mod.phase_ledger(tr, B, oracle_mod.EVICT_OPT)
    bound = sum(max(c / 2.0, 1.0) for c in lru[1:-1, 3])   # complete phases only
    assert float(opt[1:, 1].sum()) >= bound - 1.0
