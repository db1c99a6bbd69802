"""Seeded synthetic input generators (raw traces) shared by the CUDA path and the oracle.

This module holds NONE of the method's arithmetic: no block-identity chaining,
no hashing, no routing or eviction.  It only draws per-block content keys,
lengths, output sizes and arrival times, shaped like the paper's workloads
(App. A "Workloads").  Both the CUDA path
(``kvr_trace_load``) and the CPU oracle (``kvro_chain`` / ``kvro_run``)
consume the same ``RawTrace``; each side chains the keys itself.

Recipes (token lengths scaled x1/4 so that a 512-block cache holds tens of queries,
as the paper's 200k-token cache does):

* ``gsp``    Generated Shared Prefix: group g has length
             {128,256,512,1024,2048}[g mod 5] tokens, the first
             floor(ceil(r*len)/16) blocks shared by the group, the rest unique.
* ``mt``     multi-turn (ShareGPT / UltraChat shaped): client c has
             {2,4,6,8}[c mod 4] rounds; all clients share a floor(32*r)-block
             system prompt; round k's input is the previous complete path plus
             16 new blocks (256 tokens); rounds stay in order, clients interleave.
* ``ld``     long-document QA (Loogle shaped): doc d has
             {256,512,1024,2048}[d mod 4] tokens; Q_d questions of 4 unique
             blocks each.
* ``drift``  drifting popularity (config 3, "evolving patterns" P:10): group
             rank ~ Zipf(s) over G groups, the rank->group map rotates by G/64
             every N/64 queries; GSP-style members with r = 0.5.
* ``adv``    Thm 1 lower-bound family: B-L+2 paths sharing an
             (L-1)-block prefix with distinct tail blocks, queried cyclically.
* ``adv_rand`` Thm 5 family: tails drawn uniformly.

Every query carries one unique output block and |a| = 4 tokens (P:394,
P:632), except the adversarial families (no output, |a| = 0).  Arrivals are
Poisson with rate lambda = util*W / ((alpha_miss*E|q| +
o*|a|)/1000) req/s so the all-miss utilisation is ``util`` (proposed reading,
DESIGN.md §4); gaps accumulate in fp64 here and are an INPUT to both paths.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

BLOCK_TOKENS = 16
GSP_LENGTHS = (128, 256, 512, 1024, 2048)
LD_LENGTHS = (256, 512, 1024, 2048)
MT_ROUNDS = (2, 4, 6, 8)


@dataclass
class RawTrace:
    name: str
    block_tokens: int
    hash_salt: int
    arrival_ms: np.ndarray      # f64 [N], nondecreasing
    n_in_blocks: np.ndarray     # u32 [N]
    n_out_blocks: np.ndarray    # u32 [N]
    out_tokens: np.ndarray      # u32 [N]
    block_offsets: np.ndarray   # u64 [N+1]
    block_keys: np.ndarray      # u64 [sum n]

    @property
    def n_queries(self) -> int:
        return int(len(self.n_in_blocks))

    @property
    def total_blocks(self) -> int:
        return int(self.block_offsets[-1])

    @property
    def max_blocks(self) -> int:
        if self.n_queries == 0:
            return 0
        return int((self.n_in_blocks.astype(np.int64) + self.n_out_blocks).max())

    def prefix(self, n: int) -> "RawTrace":
        """The first n queries (same arrivals)."""
        n = min(n, self.n_queries)
        off = self.block_offsets[: n + 1].copy()
        return RawTrace(self.name + f"[:{n}]", self.block_tokens, self.hash_salt,
                        self.arrival_ms[:n].copy(), self.n_in_blocks[:n].copy(),
                        self.n_out_blocks[:n].copy(), self.out_tokens[:n].copy(), off,
                        self.block_keys[: int(off[-1])].copy())


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed))


def _u64(rng: np.random.Generator, n) -> np.ndarray:
    return rng.integers(0, 2 ** 64, size=n, dtype=np.uint64, endpoint=False)


def poisson_arrivals(rng: np.random.Generator, n: int, rate_per_s: Optional[float]) -> np.ndarray:
    if n == 0:
        return np.zeros(0, dtype=np.float64)
    if rate_per_s is None or rate_per_s <= 0:
        return np.zeros(n, dtype=np.float64)
    u = rng.random(n)
    gaps = -np.log1p(-u) / rate_per_s * 1000.0
    return np.cumsum(gaps).astype(np.float64)


def utilisation_rate(n_in_blocks: np.ndarray, out_tokens: np.ndarray, W: int, util: float = 0.8,
                     alpha_miss_ms: float = 1.0, out_ms_per_token: float = 20.0,
                     block_tokens: int = BLOCK_TOKENS) -> float:
    """lambda (req/s) that loads W all-miss servers to ``util``."""
    mean_service_ms = (alpha_miss_ms * float(np.mean(n_in_blocks)) * block_tokens
                       + out_ms_per_token * float(np.mean(out_tokens)))
    return util * W / (mean_service_ms / 1000.0)


def _assemble(name, n_in, n_out, out_tokens, keys, arrival, salt=0) -> RawTrace:
    n_in = np.asarray(n_in, dtype=np.uint32)
    n_out = np.asarray(n_out, dtype=np.uint32)
    off = np.zeros(len(n_in) + 1, dtype=np.uint64)
    np.cumsum(n_in.astype(np.uint64) + n_out, out=off[1:])
    assert int(off[-1]) == len(keys)
    return RawTrace(name, BLOCK_TOKENS, salt, np.asarray(arrival, dtype=np.float64), n_in, n_out,
                    np.asarray(out_tokens, dtype=np.uint32), off,
                    np.ascontiguousarray(keys, dtype=np.uint64))


def _shared_prefix_keys(rng, group, n_in, shared, n_groups, with_output=True):
    """Keys for queries whose first shared[q] blocks are the prefix of their group."""
    n_out = np.ones_like(n_in) if with_output else np.zeros_like(n_in)
    n = n_in.astype(np.int64) + n_out
    total = int(n.sum())
    keys = _u64(rng, total)                                   # unique by default
    max_sp = int(shared.max()) if len(shared) else 0
    if max_sp > 0:
        table = _u64(rng, (n_groups, max_sp))
        starts = np.zeros(len(n), dtype=np.int64)
        np.cumsum(n[:-1], out=starts[1:])
        q_of = np.repeat(np.arange(len(n)), n)
        pos = np.arange(total) - starts[q_of]
        mask = pos < shared[q_of]
        keys[mask] = table[group[q_of[mask]], pos[mask]]
    return keys, n_out


def gsp(groups: int, per_group: int, ratio: float, seed: int, order: str = "random",
        W: int = 4, util: float = 0.8, rate_per_s: Optional[float] = None,
        lengths: Sequence[int] = GSP_LENGTHS, out_tokens: int = 4) -> RawTrace:
    rng = _rng(seed)
    g_len = np.array([lengths[g % len(lengths)] for g in range(groups)], dtype=np.int64)
    g_in = g_len // BLOCK_TOKENS
    g_sp = np.ceil(ratio * g_len).astype(np.int64) // BLOCK_TOKENS   # A1 rounding
    if order == "random":
        group = np.repeat(np.arange(groups), per_group)
        group = group[rng.permutation(len(group))]
    elif order == "rr":   # worst-case round-robin over groups
        group = np.tile(np.arange(groups), per_group)
    else:
        raise ValueError(order)
    n_in = g_in[group]
    keys, n_out = _shared_prefix_keys(rng, group, n_in, g_sp[group], groups)
    ot = np.full(len(group), out_tokens, dtype=np.uint32)
    rate = rate_per_s if rate_per_s is not None else utilisation_rate(n_in, ot, W, util)
    arr = poisson_arrivals(rng, len(group), rate)
    return _assemble(f"gsp(G={groups},Q={per_group},r={ratio},{order})", n_in, n_out, ot, keys, arr)


def ld(docs: int, questions: int, seed: int, W: int = 4, util: float = 0.8,
       q_blocks: int = 4, lengths: Sequence[int] = LD_LENGTHS, out_tokens: int = 4,
       order: str = "random") -> RawTrace:
    rng = _rng(seed)
    d_blocks = np.array([lengths[d % len(lengths)] // BLOCK_TOKENS for d in range(docs)])
    if order == "random":
        group = np.repeat(np.arange(docs), questions)
        group = group[rng.permutation(len(group))]
    else:
        group = np.tile(np.arange(docs), questions)
    n_in = d_blocks[group] + q_blocks
    keys, n_out = _shared_prefix_keys(rng, group, n_in, d_blocks[group], docs)
    ot = np.full(len(group), out_tokens, dtype=np.uint32)
    arr = poisson_arrivals(rng, len(group), utilisation_rate(n_in, ot, W, util))
    return _assemble(f"ld(D={docs},Q={questions})", n_in, n_out, ot, keys, arr)


def mt(clients: int, ratio: float, seed: int, W: int = 4, util: float = 0.8,
       user_blocks: int = 16, out_tokens: int = 4, rounds: Sequence[int] = MT_ROUNDS,
       name: str = "mt") -> RawTrace:
    rng = _rng(seed)
    sp = int(np.floor(32 * ratio))
    sys_keys = _u64(rng, sp)
    R = np.array([rounds[c % len(rounds)] for c in range(clients)], dtype=np.int64)
    # each client's conversation: sys prompt, then (user_blocks user, 1 output) per round
    conv = [np.concatenate([sys_keys, _u64(rng, int(R[c]) * (user_blocks + 1))])
            for c in range(clients)]
    seq = np.repeat(np.arange(clients), R)
    seq = seq[rng.permutation(len(seq))]
    seen = np.zeros(clients, dtype=np.int64)
    n_in, parts = [], []
    for c in seq:
        k = seen[c] + 1
        seen[c] = k
        ni = sp + user_blocks * k + (k - 1)
        n_in.append(ni)
        parts.append(conv[c][: ni + 1])            # input + this round's output block
    n_in = np.array(n_in, dtype=np.int64)
    keys = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint64)
    ot = np.full(len(seq), out_tokens, dtype=np.uint32)
    arr = poisson_arrivals(rng, len(seq), utilisation_rate(n_in, ot, W, util))
    return _assemble(f"{name}(C={clients},r={ratio})", n_in, np.ones_like(n_in), ot, keys, arr)


def drift(groups: int, n_queries: int, seed: int, s: float = 1.1, W: int = 16,
          util: float = 0.8, ratio: float = 0.5, lengths: Sequence[int] = GSP_LENGTHS,
          out_tokens: int = 4) -> RawTrace:
    rng = _rng(seed)
    w = 1.0 / np.arange(1, groups + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rank = np.searchsorted(cdf, rng.random(n_queries), side="right")
    rank = np.minimum(rank, groups - 1)
    period = max(1, n_queries // 64)
    shift = (np.arange(n_queries) // period) * max(1, groups // 64)
    group = (rank + shift) % groups
    g_len = np.array([lengths[g % len(lengths)] for g in range(groups)], dtype=np.int64)
    g_in = g_len // BLOCK_TOKENS
    g_sp = np.ceil(ratio * g_len).astype(np.int64) // BLOCK_TOKENS
    n_in = g_in[group]
    keys, n_out = _shared_prefix_keys(rng, group, n_in, g_sp[group], groups)
    ot = np.full(n_queries, out_tokens, dtype=np.uint32)
    arr = poisson_arrivals(rng, n_queries, utilisation_rate(n_in, ot, W, util))
    return _assemble(f"drift(G={groups},N={n_queries},s={s})", n_in, n_out, ot, keys, arr)


def adv(B: int, L: int, cycles: int, seed: int = 0, rate_per_s: Optional[float] = None,
        util: float = 0.8) -> RawTrace:
    """Thm 1 construction: B-L+2 paths, shared (L-1)-block prefix."""
    assert 2 <= L <= B
    rng = _rng(seed)
    npaths = B - L + 2
    prefix = _u64(rng, L - 1)
    tails = _u64(rng, npaths)
    idx = np.tile(np.arange(npaths), cycles)
    return _adv_from_idx(f"adv(B={B},L={L},cycles={cycles})", prefix, tails, idx, rng, L,
                         rate_per_s, util)


def adv_rand(B: int, L: int, n: int, seed: int, rate_per_s: Optional[float] = None,
             util: float = 0.8) -> RawTrace:
    """Thm 5 construction: each query's tail uniform over B-L+2."""
    rng = _rng(seed)
    npaths = B - L + 2
    prefix = _u64(rng, L - 1)
    tails = _u64(rng, npaths)
    idx = rng.integers(0, npaths, size=n)
    return _adv_from_idx(f"adv_rand(B={B},L={L},n={n})", prefix, tails, idx, rng, L,
                         rate_per_s, util)


def _adv_from_idx(name, prefix, tails, idx, rng, L, rate_per_s, util):
    n = len(idx)
    keys = np.empty(n * L, dtype=np.uint64)
    keys.reshape(n, L)[:, : L - 1] = prefix
    keys.reshape(n, L)[:, L - 1] = tails[idx]
    n_in = np.full(n, L, dtype=np.uint32)
    ot = np.zeros(n, dtype=np.uint32)
    rate = rate_per_s if rate_per_s is not None else utilisation_rate(n_in, ot, 1, util)
    arr = poisson_arrivals(rng, n, rate)
    return _assemble(name, n_in, np.zeros(n, dtype=np.uint32), ot, keys, arr)


def random_tree(n_queries: int, seed: int, max_len: int = 6, alphabet: int = 3,
                max_out: int = 1, W: int = 2, util: float = 0.8, zero_arrivals: bool = False,
                out_tokens_max: int = 4) -> RawTrace:
    """Small random prefix-sharing traces for tests: block keys from a tiny
    alphabet so that paths share prefixes often (brute force / invariants)."""
    rng = _rng(seed)
    n_in = rng.integers(1, max_len + 1, size=n_queries)
    n_out = rng.integers(0, max_out + 1, size=n_queries)
    n = n_in + n_out
    keys = rng.integers(0, alphabet, size=int(n.sum())).astype(np.uint64)
    ot = rng.integers(0, out_tokens_max + 1, size=n_queries).astype(np.uint32)
    if zero_arrivals:
        arr = np.zeros(n_queries)
    else:
        arr = poisson_arrivals(rng, n_queries, utilisation_rate(n_in, ot, W, util))
    return _assemble(f"random_tree(n={n_queries},seed={seed})", n_in, n_out, ot, keys, arr)


def from_paths(paths: Sequence[Sequence[int]], n_out: Optional[Sequence[int]] = None,
               arrival_ms: Optional[Sequence[float]] = None,
               out_tokens: Optional[Sequence[int]] = None, name: str = "paths",
               block_tokens: int = BLOCK_TOKENS) -> RawTrace:
    """Explicit trace: paths[j] = content keys of Gamma_j (input then output)."""
    N = len(paths)
    n_out = np.zeros(N, dtype=np.uint32) if n_out is None else np.asarray(n_out, dtype=np.uint32)
    n_tot = np.array([len(p) for p in paths], dtype=np.int64)
    n_in = n_tot - n_out
    keys = np.array([k for p in paths for k in p], dtype=np.uint64)
    arr = np.zeros(N) if arrival_ms is None else np.asarray(arrival_ms, dtype=np.float64)
    ot = np.zeros(N, dtype=np.uint32) if out_tokens is None else np.asarray(out_tokens, np.uint32)
    tr = _assemble(name, n_in, n_out, ot, keys, arr)
    tr.block_tokens = block_tokens
    return tr
