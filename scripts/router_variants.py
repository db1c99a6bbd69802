"""Router variants on the GPU: the two readings of LBGR's "learning
rate 0.992" (A8 NLMS step vs A8b RLS forgetting factor), the decay-interval
ablation of P:791-795 (Delta t = 10..80 ms and no decay), the approximate / stale
global tracker (§8f #3, App. E, reading A29), and the baselines, on
config 2's GSP shape (W = 8) and config 3's drifting trace (W = 16).  RLT eviction;
`trials` seeded trials per cell, all cells in one multi-trial launch.

usage: python scripts/router_variants.py [queries=20000] [trials=32] [out.json]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import (ROUTE_LBGR, ROUTE_LBGR_RLS, ROUTE_RANDOM,  # noqa: E402
                                       ROUTE_ROUND_ROBIN, ROUTE_STATIC_LINEAR, ROUTE_THRESHOLD,
                                       DeviceTrace, Policy, Simulator, policies_array)

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 32
out_path = sys.argv[3] if len(sys.argv) > 3 else None

CELLS = [("LBGR NLMS (A8), dt=10", dict(router=ROUTE_LBGR, delta_t_ms=10.0)),
         ("LBGR NLMS (A8), dt=20 (App. A)", dict(router=ROUTE_LBGR, delta_t_ms=20.0)),
         ("LBGR NLMS (A8), dt=40", dict(router=ROUTE_LBGR, delta_t_ms=40.0)),
         ("LBGR NLMS (A8), dt=80", dict(router=ROUTE_LBGR, delta_t_ms=80.0)),
         ("LBGR NLMS (A8), no decay", dict(router=ROUTE_LBGR, delta_t_ms=math.inf)),
         ("LBGR RLS (A8b), dt=10", dict(router=ROUTE_LBGR_RLS, delta_t_ms=10.0)),
         ("LBGR RLS (A8b), dt=20 (App. A)", dict(router=ROUTE_LBGR_RLS, delta_t_ms=20.0)),
         ("LBGR RLS (A8b), dt=40", dict(router=ROUTE_LBGR_RLS, delta_t_ms=40.0)),
         ("LBGR RLS (A8b), dt=80", dict(router=ROUTE_LBGR_RLS, delta_t_ms=80.0)),
         ("LBGR RLS (A8b), no decay", dict(router=ROUTE_LBGR_RLS, delta_t_ms=math.inf)),
         ("LBGR RLS dt=20, tracker lag 1", dict(router=ROUTE_LBGR_RLS, tracker_lag=1)),
         ("LBGR RLS dt=20, tracker grain 8", dict(router=ROUTE_LBGR_RLS, tracker_grain=8)),
         ("LBGR RLS dt=20, tracker grain 32", dict(router=ROUTE_LBGR_RLS, tracker_grain=32)),
         ("LBGR RLS dt=20, lag 1 + grain 32", dict(router=ROUTE_LBGR_RLS, tracker_lag=1, tracker_grain=32)),
         ("LBGR NLMS dt=40, tracker lag 1", dict(router=ROUTE_LBGR, delta_t_ms=40.0, tracker_lag=1)),
         ("LBGR NLMS dt=40, tracker grain 32", dict(router=ROUTE_LBGR, delta_t_ms=40.0, tracker_grain=32)),
         ("Static linear (A17)", dict(router=ROUTE_STATIC_LINEAR)),
         ("Static linear, tracker grain 32", dict(router=ROUTE_STATIC_LINEAR, tracker_grain=32)),
         ("Threshold / cache-aware (A16)", dict(router=ROUTE_THRESHOLD)),
         ("Round robin", dict(router=ROUTE_ROUND_ROBIN)),
         ("Random", dict(router=ROUTE_RANDOM))]

WORKLOADS = [("config-2 GSP r=0.5, W=8", 8, lambda: wl.gsp(125, max(1, nq // 125), 0.5, seed=0xC3, W=8,
                                                          util=0.4, lengths=(128, 256, 512, 1024, 2048))),
             ("config-3 DRIFT, W=16", 16, lambda: wl.drift(8192, 1_000_000, seed=0xC5, W=16).prefix(nq))]

rows = []
for wname, W, make in WORKLOADS:
    tr = make()
    dt = DeviceTrace(tr)
    pols, keys, cell_of = [], [], []
    for c, (_, kw) in enumerate(CELLS):
        for t in range(K):
            pols.append(Policy(eviction=1, **kw))
            keys.append(1 + 1000 * c + t)
            cell_of.append(c)
    sim = Simulator(W, 512, pending_ring=1 << 15)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = sim.run(dt, np.asarray(keys, np.uint64), policies_array(pols))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res = out.results
    cell_of = np.asarray(cell_of)
    for c, (cname, _) in enumerate(CELLS):
        r = res[cell_of == c]
        ok = r["status"] == 0
        q = r["queries"].astype(np.float64)
        lat = r["sum_latency_ms"] / q
        ttft = r["sum_ttft_ms"] / q
        hit = r["hit_tokens"] / r["input_tokens"]
        mk = r["makespan_ms"]
        row = {"workload": wname, "router": cname, "trials_ok": int(ok.sum()), "trials": len(r),
               "mean_latency_ms": float(lat.mean()), "latency_se": float(lat.std() / math.sqrt(len(r))),
               "mean_ttft_ms": float(ttft.mean()), "ttft_se": float(ttft.std() / math.sqrt(len(r))),
               "hit_rate": float(hit.mean()), "makespan_ms": float(mk.mean()), "launch_ms": ms}
        rows.append(row)
        print(json.dumps(row), flush=True)

print()
print("| workload | router | mean latency (ms) | mean TTFT (ms) | hit rate | makespan (ms) |")
print("|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['workload']} | {r['router']} | {r['mean_latency_ms']:.1f} ± {r['latency_se']:.1f} | "
          f"{r['mean_ttft_ms']:.1f} ± {r['ttft_se']:.1f} | {r['hit_rate']:.3f} | {r['makespan_ms']:.0f} |")
if out_path:
    with open(out_path, "w") as f:
        json.dump(rows, f, indent=1)
