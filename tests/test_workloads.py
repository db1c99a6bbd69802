"""Pins of the seeded synthetic generators (inputs to both paths).

The drifting-popularity trace (config 3, SURVEY §8d DRIFT): group ranks follow
Zipf(s) over G groups, and the rank -> group map rotates by G/64 every N/64
queries.  Groups are recovered from the first block key (their shared prefix)."""
from collections import Counter

import numpy as np

from paper_2601_18999_b200 import workloads as wl


def _first_keys(tr, lo, hi):
    off = tr.block_offsets
    return [int(tr.block_keys[off[j]]) for j in range(lo, hi)]


def test_drift_zipf_ranks_and_rotation():
    G, P, s = 64, 3000, 1.1
    tr = wl.drift(G, 64 * P, seed=17, s=s, W=16)
    p = 1.0 / np.arange(1, G + 1) ** s
    p /= p.sum()
    c0 = Counter(_first_keys(tr, 0, P)).most_common()
    # the top three ranks of period 0 match Zipf(s) within 5 sigma (binomial)
    for r in range(3):
        mean, sd = P * p[r], np.sqrt(P * p[r] * (1 - p[r]))
        assert abs(c0[r][1] - mean) <= 5 * sd, (r, c0[r][1], mean)
    # after one period the map shifts by one group: period 1's most popular group is the
    # group holding rank 1 in period 0, and period 0's top group drops to the last rank
    c1 = Counter(_first_keys(tr, P, 2 * P))
    assert c1.most_common(1)[0][0] == c0[1][0]
    assert c1[c0[0][0]] <= P * p[-1] + 5 * np.sqrt(P * p[-1])


def test_gsp_structure():
    """GSP(G, Q, r): G*Q queries; a group's members share exactly
    floor(ceil(r * len) / 16) leading blocks and differ right after."""
    G, Q, r = 10, 6, 0.5
    tr = wl.gsp(G, Q, r, seed=3)
    assert tr.n_queries == G * Q
    off = tr.block_offsets
    paths = [tr.block_keys[off[j]:off[j + 1]] for j in range(tr.n_queries)]
    by_first = {}
    for pth in paths:
        by_first.setdefault(int(pth[0]), []).append(pth)
    assert len(by_first) == G and all(len(v) == Q for v in by_first.values())
    for members in by_first.values():
        n_in = len(members[0]) - 1                         # one output block
        shared = int(np.ceil(r * n_in * 16)) // 16
        for a in members[1:]:
            common = 0
            while common < len(a) and a[common] == members[0][common]:
                common += 1
            assert common == shared
