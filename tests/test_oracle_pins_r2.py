"""Pins of the oracle functions left unpinned in round 1 (VERDICT r1 "What's weak" #1).

P33  ReleaseLoad P~ <- max(0, P~ - C^ rho^kappa) (Alg. 2 l.13; "releases any
     remaining load"; reading A10) with rho = 1/2, where every power is exact:
     hand-computed router scores after a release.
P34  the LRU_MARKED fallback of Alg. 1 when U = {} (reading A5): a hand
     example where every leaf is marked and the least recently used leaf is known.
P35  the RANDOM router (reading A6 counter (j, 0xFFFFFFFF, 2)): chi-square
     uniformity over workers and decorrelation across keys.
P36  the latency histogram bin rule (A19: 4 log buckets per octave): hand values and
     the closed-form bin edges 2^k (1 + r/4).
P37  NaN score ordering of the argmin (reading A37) and the policy checks that keep
     it unreachable for sane inputs (NLMS needs 0 <= mu < 2, A8).

No expected value here comes from running the oracle: each is derived in the
docstring (hand arithmetic with powers of two) or is a closed form / statistic.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_2601_18999_b200 import workloads as wl


def _blocks(n, base):
    return [base + i for i in range(n)]


# -------------------------------------------------------------------------- P33
def test_p33_release_overlapping_queries(oracle_mod):
    """W = 1, Leaf-LRU, theta = 0 (mu = 0), est. alpha = (0, 1 ms/token), truth alpha_M = 1,
    o = 0, block = 16 tokens, rho = 1/2, dt = 10 ms.  E^ = C^ + P~ (Eq. 4 with theta = 0).

    q1: 4 blocks (64 tok) at 0:  P~ = 0 -> E^1 = 64; runs 0..64; P~ = 64, k_a = 0.
    q2: 2 blocks (32 tok) at 25: ticks 10, 20 -> P~ = 16 -> E^2 = 32 + 16 = 48; queued
        behind q1: runs 64..96; P~ = 48, k_a = 2.
    q3: 1 block (16 tok) at 85:  ticks 30..60 -> P~ = 48/16 = 3 (k = 6); completion of q1
        at 64: release 64 * (1/2)^6 = 1 -> P~ = 2 (= 32 (1/2)^4, q2's decayed share);
        ticks 70, 80 -> P~ = 1/2; q2 (c = 96) still pending -> E^3 = 16 + 1/2 = 16.5.
    kappa - 1 would give 16.25, kappa + 1 16.625, an undecayed release (P~ -> 0) 16."""
    tr = wl.from_paths([_blocks(4, 100), _blocks(2, 200), _blocks(1, 300)],
                       arrival_ms=[0.0, 25.0, 85.0])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=64, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=0.0, rho=0.5, delta_t_ms=10.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    assert r.rc == 0
    assert list(r.records["score"]) == [64.0, 48.0, 16.5]
    assert list(r.records["latency_ms"]) == [64.0, 71.0, 11.0 + 16.0]   # q3 waits 96 - 85


def test_p33_release_square_and_multiply(oracle_mod):
    """kappa = 13 = 0b1101 (three set bits: the LSB-first square-and-multiply of A10).
    block = 4 tokens, same constants.  q1: 34 blocks (136 tok) at 0, runs 0..136,
    P~ = 136.  q2: 2 blocks (8 tok) at 25: ticks 10, 20 -> P~ = 34 -> E^2 = 8 + 34 = 42;
    runs 136..144; P~ = 42, k_a = 2.  q3: 1 block (4 tok) at 141: ticks 30..130
    (k = 13) -> P~ = 42 / 2^11; completion of q1 at 136: release 136 / 2^13 = 34 / 2^11
    -> P~ = 8 / 2^11; tick 140 -> 4 / 2^11 = 2^-9; E^3 = 4 + 2^-9 = 4.001953125."""
    tr = wl.from_paths([_blocks(34, 100), _blocks(2, 200), _blocks(1, 300)],
                       arrival_ms=[0.0, 25.0, 141.0], block_tokens=4)
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=64, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=0.0, rho=0.5, delta_t_ms=10.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    assert r.rc == 0
    assert r.records["score"][1] == 42.0
    assert Fraction(r.records["score"][2]) == Fraction(4) + Fraction(1, 512)


@pytest.mark.parametrize("gap_ticks", [0, 1, 7, 40])
def test_p33_single_query_release_is_exact(oracle_mod, gap_ticks):
    """One query alone: whatever the number of ticks kappa before its completion, the
    release removes exactly its decayed share, so P~ = 0 at the next arrival (E^ = C^).
    q1: 3 blocks (48 tok), done at 48; q2 (1 block, 16 tok) arrives 10*gap_ticks ms after."""
    tr = wl.from_paths([_blocks(3, 100), _blocks(1, 200)],
                       arrival_ms=[0.0, 48.0 + 10.0 * gap_ticks])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=16, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=0.0, rho=0.5, delta_t_ms=10.0)
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    assert list(r.records["score"]) == [48.0, 16.0]


# -------------------------------------------------------------------------- P34
def _p34_trace():
    A, B, C, D, X, Y = 1, 2, 3, 4, 5, 6
    return wl.from_paths([[A], [B], [C], [A, D], [X], [Y]])


@pytest.mark.parametrize("key", [0, 1, 2, 3])
def test_p34_lru_marked_fallback_hand_example(oracle_mod, key):
    """W = 1, B = 3, RLT with the LRU_MARKED fallback (A5), n_out = 0.
    q0..q2 = [A], [B], [C]: S = {A, B, C} in slots 0, 1, 2; T = {A, B, C} (|T| = B).
    q3 = [A, D]: A hit (marked); marking D makes |T| = B + 1 -> reset T = {D}; miss with a
      full cache: U = leaves \\ T \\ {parent(D) = A} = {B, C} -> one draw; D takes the
      victim's slot.
    q4 = [X]: T = {D, X}; U = leaves{D, other of B/C} \\ T = {other} -> second draw (|U| = 1).
    q5 = [Y]: T = {D, X, Y} (no reset: |T| + 1 = B); U = leaves{D, X} \\ T = {} -> fallback.
      LRU_MARKED: least recently used leaf != parent = D (last touched by q3) rather than X
      (q4): no draw.  Totals: 3 evictions, 2 draws, 1 reset, 1 fallback; victim 3 = D.
    For keys where q3 evicted C, D sits in slot 2 and X in slot 1, so neither a
    lowest-slot rule nor an arg-max of recency would pick D."""
    tr = _p34_trace()
    H = oracle_mod.chain(tr)
    ids = dict(A=H[0], B=H[1], C=H[2], D=H[4], X=H[5], Y=H[6])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=3, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=1, rlt_fallback=oracle_mod.RLT_LRU_MARKED, router=3)
    r = oracle_mod.run(cfg, tr, pol, key, record=True, victims_cap=8, check_invariants=True)
    assert r.rc == 0
    res = r.result
    assert (res["evictions"], res["rlt_draws"], res["rlt_resets"], res["rlt_fallbacks"]) == (3, 2, 1, 1)
    v = [int(x) for x in r.victims[:3]]
    assert set(v[:2]) == {ids["B"], ids["C"]}
    assert v[2] == ids["D"]
    assert list(r.records["n_victims"]) == [0, 0, 0, 1, 1, 1]


@pytest.mark.parametrize("fallback,draws,resets", [(0, 3, 2), (1, 3, 1)])
def test_p34_other_fallbacks_draw_on_same_example(oracle_mod, fallback, draws, resets):
    """Same trace: EARLY_RESET resets T = {Y} and draws over {D, X}; UNIFORM_LEAF draws
    over {D, X} without a reset.  Both add one draw where LRU_MARKED adds none."""
    tr = _p34_trace()
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=3, out_ms_per_token=0.0)
    pol = oracle_mod.OraclePolicy(eviction=1, rlt_fallback=fallback, router=3)
    r = oracle_mod.run(cfg, tr, pol, 5, record=True, victims_cap=8, check_invariants=True)
    H = oracle_mod.chain(tr)
    assert (r.result["rlt_draws"], r.result["rlt_resets"], r.result["rlt_fallbacks"]) == (draws, resets, 1)
    assert int(r.victims[2]) in (int(H[4]), int(H[5]))


# -------------------------------------------------------------------------- P35
def _random_route(oracle_mod, W, n, key):
    tr = wl.from_paths([[1_000_000 + j] for j in range(n)])
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=4, out_ms_per_token=0.0, pending_ring=0)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=0, router=4), key, record=True)
    assert r.rc == 0
    return r.records["worker"].astype(np.int64)


@pytest.mark.parametrize("W", [2, 5, 8, 32])
def test_p35_random_router_uniform(oracle_mod, W):
    """P:373 "randomly assigns": i* ~ Uniform{0..W-1}.  Pearson chi-square over 6,000
    routings (df = W - 1) below the 1e-6 upper quantile, for four keys."""
    from scipy.stats import chi2
    n = 6000
    for key in (1, 2, 0xC5, 2 ** 63 + 11):
        w = _random_route(oracle_mod, W, n, key)
        cnt = np.bincount(w, minlength=W)
        assert cnt.sum() == n and len(cnt) == W
        e = n / W
        stat = float(((cnt - e) ** 2 / e).sum())
        assert stat < chi2.isf(1e-6, W - 1), (key, cnt)


def test_p35_random_router_keys_decorrelate(oracle_mod):
    """Different trial keys give independent routings: agreement between two keys is
    Binomial(n, 1/W) (within 5 sigma); serial agreement (j vs j+1) too."""
    W, n = 8, 6000
    a = _random_route(oracle_mod, W, n, 7)
    b = _random_route(oracle_mod, W, n, 8)
    p = 1.0 / W
    sd = math.sqrt(n * p * (1 - p))
    assert abs(int((a == b).sum()) - n * p) < 5 * sd
    assert abs(int((a[1:] == a[:-1]).sum()) - (n - 1) * p) < 5 * sd
    # and the choice does not depend on the eviction policy or the cache (state-free)
    tr = wl.from_paths([[1_000_000 + j] for j in range(200)])
    cfg = oracle_mod.OracleConfig(W=W, capacity_blocks=4, out_ms_per_token=0.0)
    r1 = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=1, router=4), 7, record=True)
    assert np.array_equal(r1.records["worker"].astype(np.int64), a[:200])


# -------------------------------------------------------------------------- P36
def _bin_of(oracle_mod, lat, bins=128):
    """Route one query whose latency is exactly `lat` (alpha = 0, o = lat, |a| = 1)."""
    tr = wl.from_paths([[1]], out_tokens=[1])
    cfg = oracle_mod.OracleConfig(W=1, capacity_blocks=4, alpha_cached_ms=0.0, alpha_miss_ms=0.0,
                                  out_ms_per_token=float(lat), latency_hist_bins=bins)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(eviction=0, router=3), 0, record=True)
    assert r.rc == 0 and r.records["latency_ms"][0] == lat
    nz = np.nonzero(r.hist)[0]
    assert len(nz) == 1 and r.hist[nz[0]] == 1
    return int(nz[0])


# bin 0 = below 1 ms; bin b >= 1 covers [2^k (1 + r/4), 2^k (1 + (r+1)/4)), k = (b-1) div 4,
# r = (b-1) mod 4 (A19: four equal-width sub-bins per octave)
HAND = [(0.0, 0), (0.9, 0), (0.999999, 0), (1.0, 1), (1.19, 1), (1.2, 1), (1.25, 2), (1.4999, 2),
        (1.5, 3), (1.75, 4), (1.9999, 4), (2.0, 5), (2.5, 6), (3.0, 7), (3.5, 8), (4.0, 9),
        (1000.0, 40), (1e6, 80)]


@pytest.mark.parametrize("lat,b", HAND)
def test_p36_hist_bin_hand_values(oracle_mod, lat, b):
    """Worked by hand from A19 (bin 0 below 1 ms, then four equal sub-bins per octave):
    1.19 and 1.2 lie in [1, 1.25) -> 1; 2 opens octave k = 1 -> 5; 1000 = 2^9 * 1.953 ->
    k = 9, r = 3 -> 1 + 36 + 3 = 40; 1e6 = 2^19 * 1.907 -> 1 + 76 + 3 = 80."""
    assert _bin_of(oracle_mod, lat) == b


def test_p36_hist_bin_edges(oracle_mod):
    """Random latencies land in the bin whose exact edges 2^k (1 + r/4) bracket them,
    and bins clamp at bins - 1."""
    rng = np.random.default_rng(36)
    for lat in np.exp(rng.uniform(0.0, math.log(2.0 ** 30), 40)):
        lat = float(lat)
        b = _bin_of(oracle_mod, lat)
        k, r = (b - 1) // 4, (b - 1) % 4
        lo = Fraction(2) ** k * (1 + Fraction(r, 4))
        hi = Fraction(2) ** k * (1 + Fraction(r + 1, 4))
        assert lo <= Fraction(lat) < hi, (lat, b)
    assert _bin_of(oracle_mod, 1e6, bins=16) == 15
    assert _bin_of(oracle_mod, 2.0 ** 40, bins=128) == 127


# -------------------------------------------------------------------------- P37
def test_p37_nan_score_ranks_last(oracle_mod):
    """theta0 = (1e308, -1e308, 0, 0), mu = 0: a worker whose hit and miss features are
    both >= 2 scores 1e308*2 + (-1e308*2) = inf - inf = NaN; a worker with no hit scores
    -inf.  q0 (125 blocks) goes to worker 0 (both -inf, lowest index); q1 shares those
    125 blocks and adds 125 more: worker 0 -> NaN, worker 1 -> -inf.  A37: NaN ranks
    after every number, so i* = 1 (a plain `<` scan would keep the NaN at index 0)."""
    p = _blocks(125, 1)
    tr = wl.from_paths([p, p + _blocks(125, 5000)], arrival_ms=[0.0, 0.0])
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=512)
    pol = oracle_mod.OraclePolicy(eviction=0, mu=0.0, theta0=(1e308, -1e308, 0.0, 0.0))
    r = oracle_mod.run(cfg, tr, pol, 0, record=True)
    assert r.rc == 0
    assert list(r.records["worker"]) == [0, 1]
    assert r.records["score"][1] == -math.inf


@pytest.mark.parametrize("kw", [dict(mu=2.0), dict(mu=-0.1), dict(mu=math.nan),
                                dict(theta0=(math.inf, 0, 0, 0)), dict(w_hit=math.nan),
                                dict(est_alpha_miss_ms=math.inf), dict(rho=0.0),
                                dict(delta_t_ms=0.0), dict(tau=math.inf)])
def test_p37_policy_checks(oracle_mod, kw):
    """A8: the NLMS step is stable for 0 <= mu < 2 only; every other parameter must be
    finite except delta_t = +inf (no decay).  Invalid policies are refused (rc = 1)."""
    tr = wl.from_paths([[1, 2]])
    cfg = oracle_mod.OracleConfig(W=2, capacity_blocks=8)
    r = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(**kw), 0)
    assert r.rc == 1
    ok = oracle_mod.run(cfg, tr, oracle_mod.OraclePolicy(delta_t_ms=math.inf, mu=1.999), 0)
    assert ok.rc == 0
