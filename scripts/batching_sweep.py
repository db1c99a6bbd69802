"""Continuous batching on the GPU (A30-A36): a sweep of
the per-worker batch size beta on the bench's config-2 trace (W = 8, B = 512, prefix
ratio 0.5, LBGR), RLT vs Leaf-LRU, next to the beta = 1 model of A3/A12
(batch_slots = 0, the tuned kernel).  The premise beta * L_max <= B caps
beta at 3 for the 129-block paths at B = 512; beta = 4 and 8 run at B = 1,032
(= 8 * 129).  Reports the paper's Fig. 14 quantities (hit rate, latency, TTFT
per beta) and the kernel's throughput (query-replays/s, CUDA events on the
launching stream, one full wave of trials per cell).

usage: python scripts/batching_sweep.py [queries=100000] [trials=148] [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 148
out_path = sys.argv[3] if len(sys.argv) > 3 else None

import bench  # noqa: E402  (config 2's trace recipe: the bench's r = 0.5 GSP trace)

W = bench.C2_W
tr = bench.c2_traces(nq)[1]
dt = DeviceTrace(tr)
L_max = int(tr.max_blocks)
rows = []
for beta, B in ((0, 512), (1, 512), (2, 512), (3, 512), (4, 8 * L_max), (8, 8 * L_max), (0, 8 * L_max)):
    for ev, ename in ((1, "RLT"), (0, "L-LRU")):
        sim = Simulator(W, B, pending_ring=16384, batch_slots=beta)
        keys = np.arange(1, K + 1, dtype=np.uint64)
        pols = policies_array([Policy(eviction=ev) for _ in range(K)])
        b = sim.alloc([dt], K)
        b["keys"].copy_(torch.from_numpy(keys.view(np.int64)))
        b["policies"].copy_(torch.from_numpy(np.ascontiguousarray(pols).view(np.uint8)))
        s = torch.cuda.current_stream()
        sim.launch([dt], K, b, stream=s)          # warm-up (module load, caches)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        sim.launch([dt], K, b, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        r = sim.collect(b, K).results
        ok = r["status"] == 0
        q = r["queries"].astype(np.float64)
        tier, smem, cps = sim.plan(L_max)
        rows.append(dict(
            beta=beta, model="beta=1 model (A3/A12)" if beta == 0 else "continuous batching (A30)",
            B=B, eviction=ename, trials=K, ok=int(ok.sum()),
            hit_rate=float(np.mean(r["hit_tokens"] / r["input_tokens"])),
            mean_latency_ms=float(np.mean(r["sum_latency_ms"] / q)),
            mean_ttft_ms=float(np.mean(r["sum_ttft_ms"] / q)),
            makespan_ms=float(np.mean(r["makespan_ms"])),
            max_pending=int(r["max_pending"].max()),
            evictions_per_query=float(np.mean(r["evictions"] / q)),
            gpu_ms=ms, query_replays_per_s=float(K * tr.n_queries / (ms / 1e3)),
            tier=int(tier), smem=int(smem), ctas_per_sm=int(cps)))
        print(json.dumps(rows[-1]), flush=True)
        sim.close()

if out_path:
    with open(out_path, "w") as f:
        json.dump(dict(workload=f"config-2 bench trace r=0.5 (bench.c2_traces()[1]), W={W}, {tr.n_queries} queries, LBGR (App. A)",
                       rows=rows), f, indent=1)
