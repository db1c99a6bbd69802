"""Config-4 capacity sweep on the GPU with offline OPT (KVR_EVICT_OPT, Belady):
  * Thm 1 family ADV(B, L=4, 8 cycles): misses of Leaf-LRU, RLT (mean over
    trials) and OPT, and the ratios to OPT;
  * Thm 5 random tails ADV-RAND(B, L=4): mean number of queries between
    OPT misses against the closed form (B-L+2) H_{B-L+1} (reading A28).
All replays at W = 1 (the single-cache setting of the theorems); arrivals do not
affect the cache.  Prints one JSON object per capacity and a markdown table.

usage: python scripts/competitive_ratio.py [max_log2_B=16] [rlt_trials=32] [out.json]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import (EVICT_LRU, EVICT_OPT, EVICT_RLT, ROUTE_ROUND_ROBIN,  # noqa: E402
                                       DeviceTrace, Policy, Simulator, policies_array)

maxlog = int(sys.argv[1]) if len(sys.argv) > 1 else 16
R = int(sys.argv[2]) if len(sys.argv) > 2 else 32
out_path = sys.argv[3] if len(sys.argv) > 3 else None
L, CYCLES = 4, 8


def harmonic(n):
    return sum(1.0 / k for k in range(1, n + 1))


def timed_run(sim, dt, keys, pols):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = sim.run(dt, np.asarray(keys, np.uint64), policies_array(pols))
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


rows = []
for lb in range(6, maxlog + 1):
    B = 1 << lb
    row = {"B": B, "L": L}
    # ---- Thm 1 family: cyclic tails ----
    tr = wl.adv(B, L, CYCLES, seed=0xC6)
    dt = DeviceTrace(tr).with_next_use()
    sim = Simulator(1, B, pending_ring=1 << 16)
    pols = ([Policy(eviction=EVICT_OPT, router=ROUTE_ROUND_ROBIN),
             Policy(eviction=EVICT_LRU, router=ROUTE_ROUND_ROBIN)] +
            [Policy(eviction=EVICT_RLT, router=ROUTE_ROUND_ROBIN)] * R)
    out, ms = timed_run(sim, dt, list(range(1, R + 3)), pols)
    res = out.results
    assert np.all(res["status"] == 0), res["status"]
    miss = res["inserted_blocks"].astype(np.float64)
    cold = B + 1                       # distinct blocks: L-1 prefix + B-L+2 tails
    steady = miss - cold               # misses beyond the compulsory ones
    row.update({"queries": tr.n_queries, "opt_misses": int(miss[0]), "lru_misses": int(miss[1]),
                "rlt_misses_mean": float(miss[2:].mean()), "rlt_misses_sd": float(miss[2:].std()),
                "lru_over_opt_steady": float(steady[1] / steady[0]),
                "rlt_over_opt_steady": float(steady[2:].mean() / steady[0]),
                "thm1_lru_per_phase": B - L + 2, "harmonic_B_L_1": harmonic(B - L + 1),
                "gpu_ms": ms, "query_replays_per_s": tr.n_queries * (R + 2) / (ms / 1e3)})
    # ---- Thm 5: random tails, gaps between non-compulsory OPT misses (B <= 4096:
    # the steady state needs ~ (B-L+2) H_{B-L+2} queries just to see every tail) ----
    npaths = B - L + 2
    expect = npaths * harmonic(npaths - 1)
    row.update({"opt_gap_closed_form_A28": expect, "opt_gap_mean": None, "opt_gap_se": None,
                "opt_gaps": 0, "gpu_ms_rand": 0.0})
    if B <= 4096:
        n2 = int(40 * expect) + 2 * int(npaths * harmonic(npaths))
        tr2 = wl.adv_rand(B, L, n2, seed=0xC60 + lb)
        dt2 = DeviceTrace(tr2).with_next_use()
        sim2 = Simulator(1, B, pending_ring=1 << 16, record_trials=1)
        out2, ms2 = timed_run(sim2, dt2, [1], [Policy(eviction=EVICT_OPT, router=ROUTE_ROUND_ROBIN)])
        hit = out2.records[0]["hit_tokens"][: tr2.n_queries].astype(np.int64)
        tails = np.asarray(tr2.block_keys, np.uint64).reshape(tr2.n_queries, L)[:, L - 1]
        _, first = np.unique(tails, return_index=True)
        compulsory = np.zeros(tr2.n_queries, bool)
        compulsory[first] = True
        missq = np.nonzero((hit < L * tr2.block_tokens) & ~compulsory)[0]
        gaps = np.diff(missq)
        row.update({"rand_queries": tr2.n_queries, "gpu_ms_rand": ms2, "opt_gaps": int(len(gaps)),
                    "opt_gap_mean": float(gaps.mean()) if len(gaps) else None,
                    "opt_gap_se": float(gaps.std() / math.sqrt(len(gaps))) if len(gaps) > 1 else None})
    print(json.dumps(row), flush=True)
    rows.append(row)

print()
print("| B | queries | OPT | L-LRU | RLT (mean ± sd) | steady L-LRU/OPT (Thm 1: B-L+2) | steady RLT/OPT | H_{B-L+1} | OPT gap, random tails | (B-L+2)H_{B-L+1} (A28) | GPU ms |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    gap = f"{r['opt_gap_mean']:.0f} ± {r['opt_gap_se']:.0f} (n={r['opt_gaps']})" if r["opt_gap_mean"] else "-"
    print(f"| {r['B']} | {r['queries']} | {r['opt_misses']} | {r['lru_misses']} | "
          f"{r['rlt_misses_mean']:.1f} ± {r['rlt_misses_sd']:.1f} | {r['lru_over_opt_steady']:.1f} | "
          f"{r['rlt_over_opt_steady']:.2f} | {r['harmonic_B_L_1']:.2f} | {gap} | "
          f"{r['opt_gap_closed_form_A28']:.0f} | {r['gpu_ms'] + r['gpu_ms_rand']:.0f} |")
if out_path:
    with open(out_path, "w") as f:
        json.dump(rows, f, indent=1)
