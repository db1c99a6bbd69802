"""Competitive-analysis helpers on top of the oracle (TEST INFRASTRUCTURE).

Phase partition of §3.2: the flattened block-access sequence
of the complete paths is cut into phases that each contain exactly B distinct
blocks (the last one possibly fewer).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .binding import chain


def flattened_ids(tr) -> np.ndarray:
    """Block identities in access order (Gamma_1 || Gamma_2 || ...)."""
    return chain(tr)


def phases(ids: np.ndarray, B: int) -> List[Tuple[int, int]]:
    """Greedy left-to-right split into [start, end) ranges of B distinct ids."""
    out, start, seen = [], 0, set()
    for k, v in enumerate(ids.tolist()):
        if v not in seen and len(seen) == B:
            out.append((start, k))
            start, seen = k, set()
        seen.add(v)
    if start < len(ids):
        out.append((start, len(ids)))
    return out


def misses_per_phase(miss_flags: np.ndarray, ph: List[Tuple[int, int]]) -> np.ndarray:
    return np.array([int(miss_flags[a:b].sum()) for a, b in ph], dtype=np.int64)


def harmonic(n: int) -> float:
    return sum(1.0 / k for k in range(1, n + 1))
