"""Multi-process (gloo, world size 2) tests of the sharding and summary-reduce
host logic used by multi-GPU runs (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2601_18999_b200 import dist as kd
from paper_2601_18999_b200.kvr import RESULT_DTYPE


def _fake_results(n, seed):
    rng = np.random.default_rng(seed)
    r = np.zeros(n, dtype=RESULT_DTYPE)
    for f in ("queries", "hit_tokens", "input_tokens", "probes", "inserted_blocks", "evictions",
              "rlt_draws", "rlt_resets", "rlt_fallbacks"):
        r[f] = rng.integers(0, 1 << 40, size=n, dtype=np.uint64)
    r["decision_digest"] = rng.integers(0, 2 ** 64, size=n, dtype=np.uint64, endpoint=False)
    r["status"] = (rng.random(n) < 0.1).astype(np.int32)
    return r


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    allres = _fake_results(n, 7)
    mine = kd.shard_trials(n, rank, world)
    vec = kd.summary_vector(allres[mine], trace_hash=123)
    out = kd.reduce_summary(vec)
    if rank == 0:
        q.put(out.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_trials_partition():
    for n in (0, 1, 7, 1024):
        for world in (1, 2, 3, 8):
            parts = [kd.shard_trials(n, r, world) for r in range(world)]
            allidx = np.sort(np.concatenate(parts)) if n else np.zeros(0)
            assert np.array_equal(allidx, np.arange(n))


def test_weak_scaling_keys_distinct():
    ks = np.concatenate([kd.weak_scaling_keys(1024, r) for r in range(8)])
    assert len(np.unique(ks)) == len(ks)


def test_summary_vector_fields():
    r = _fake_results(10, 1)
    v = kd.summary_vector(r, trace_hash=5).view(np.uint64)
    assert v[0] == 10 and v[1] == r["queries"].sum() and v[11] == np.count_nonzero(r["status"])
    assert v[12] == 5


def test_gloo_world2_reduce_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 37
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = kd.summary_vector(_fake_results(n, 7), trace_hash=123).view(np.uint64).copy()
    got = np.array(got, dtype=np.int64).view(np.uint64)
    ref[12] = 2 * 123          # the trace-hash slot sums one copy per rank
    assert np.array_equal(got, ref)


def test_c5_fixed_list_sharding():
    """bench.py's config-5 plan: one fixed list of trials, rank r takes (t div 2) mod N == r;
    the union over ranks is the list at every N, shares differ by at most 2 trials, and
    every rank gets both evictions (RLT on even keys t + 1, Leaf-LRU on odd)."""
    import bench
    n = 65536
    cell = bench.c5_cell_of(n)
    sizes = np.bincount(cell, minlength=48)
    assert sizes.min() >= n // 48 and sizes.max() <= n // 48 + 1
    for world in (1, 2, 3, 4, 8):
        parts = [bench.c5_shard(n, r, world) for r in range(world)]
        allt = np.sort(np.concatenate(parts))
        assert np.array_equal(allt, np.arange(n))
        lens = [len(p) for p in parts]
        assert max(lens) - min(lens) <= 2
        for p in parts:
            keys = p + 1
            assert (keys % 2 == 0).any() and (keys % 2 == 1).any()
            # balanced per cell as well: each rank's share of a cell is within 2 of n/48/world
            per = np.bincount(cell[p], minlength=48)
            assert per.max() - per.min() <= 3


def test_c5_plan_launches_cover_the_share():
    """The per-W launches of a rank hold exactly its share, longest trace first."""
    import bench

    class _T:   # stand-in traces: only n_queries matters to the plan
        def __init__(self, n):
            self.n_queries = n
    traces = {W: [_T(100 * (k + 1) + W) for k in range(12)] for W in bench.C5_WS}
    n, world = 960, 4
    for r in range(world):
        ls = bench.c5_plan(r, world, n, traces=traces)
        got = np.sort(np.concatenate([L.tids for L in ls]))
        assert np.array_equal(got, bench.c5_shard(n, r, world))
        for L in ls:
            nq = np.array([L.traces[i].n_queries for i in L.trial_trace])
            assert np.all(np.diff(nq) <= 0)
            assert np.array_equal(L.keys, (L.tids + 1).astype(np.uint64))
            assert np.array_equal(L.evict, (L.keys % 2 == 0).astype(np.uint32))
