"""Multi-GPU plumbing: trial sharding and the single summary reduce.

Trials are independent replays (no exchange inside a replay), so a run shards
them across ranks with no data-path collective.  Each rank runs its
kvr_sim_run_multi launches over its trials; at the end one
`torch.distributed.reduce` (NCCL over NVLink on a GPU box, gloo in the CPU tests)
sums an int64 vector of summary counters to rank 0.  Floating-point aggregates
stay per trial (the per-trial result buffers).

Two sharding modes are used by bench.py:
* strong scaling (config 5, the default): ONE fixed trial list, trial t on rank
  (t div 2) mod N (`bench.c5_shard`); a trial's key and policy depend on t only, so
  its result bytes are identical at every N (P20; tests/test_gpu_bench_multirank.py);
* weak scaling (config 2, `--workload c2`): every rank runs its own trials with
  distinct keys (`weak_scaling_keys`), so N-GPU runs cover a different trial set.
`shard_trials` (t mod N) is the plain strided split for other fixed lists.
"""
from __future__ import annotations

import numpy as np

SUMMARY_FIELDS = ("trials", "queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks",
                  "evictions", "rlt_draws", "rlt_resets", "rlt_fallbacks", "digest_sum",
                  "status_nonzero", "trace_hash")


def shard_trials(n_trials: int, rank: int, world: int) -> np.ndarray:
    """Strided assignment t mod world == rank (balances cells of unequal cost)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return np.arange(rank, n_trials, world, dtype=np.int64)


def weak_scaling_keys(n_per_rank: int, rank: int) -> np.ndarray:
    """Weak scaling: every rank runs its own n_per_rank trials with distinct Philox keys."""
    return (np.uint64(rank) * np.uint64(1 << 32) + np.arange(n_per_rank, dtype=np.uint64)
            + np.uint64(1))


def summary_vector(results: np.ndarray, trace_hash: int = 0) -> np.ndarray:
    """int64 counter vector of a set of kvr_trial_result rows (u64 sums wrap mod 2^64)."""
    v = np.zeros(len(SUMMARY_FIELDS), dtype=np.uint64)
    if len(results):
        v[0] = len(results)
        for i, f in enumerate(("queries", "hit_tokens", "input_tokens", "probes",
                               "inserted_blocks", "evictions", "rlt_draws", "rlt_resets",
                               "rlt_fallbacks"), start=1):
            v[i] = np.sum(results[f].astype(np.uint64), dtype=np.uint64)
        with np.errstate(over="ignore"):
            v[10] = np.sum(results["decision_digest"].astype(np.uint64), dtype=np.uint64)
        v[11] = int(np.count_nonzero(results["status"]))
    v[12] = np.uint64(trace_hash)
    return v.view(np.int64)


def summary_tensor(results_u8, n_trials: int, trace_hash: int = 0):
    """Device-side summary_vector of the raw kvr_trial_result buffer (torch uint8,
    144 B per trial): column sums of the u64 counters (wrapping), nonzero status."""
    import torch
    r64 = results_u8[: n_trials * 144].view(torch.int64).view(n_trials, 18)
    st = results_u8[: n_trials * 144].view(torch.int32).view(n_trials, 36)[:, 34]
    out = torch.zeros(len(SUMMARY_FIELDS), dtype=torch.int64, device=results_u8.device)
    out[0] = n_trials
    out[1:10] = r64[:, 0:9].sum(dim=0)
    out[10] = r64[:, 10].sum()
    out[11] = (st != 0).sum()
    out[12] = trace_hash
    return out


def reduce_summary(vec: np.ndarray, device=None, group=None) -> np.ndarray:
    """Sum the summary vectors of all ranks onto rank 0 (one collective per run);
    the trace-hash slot then holds world_size x the hash when every rank packed
    the same trace."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(vec).copy())
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(t, dst=0, group=group)
    return t.cpu().numpy()
