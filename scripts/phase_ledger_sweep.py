"""Phase ledger on the GPU: config 4's capacity sweep
(Thm 1 family ADV(B, L=4, 8 cycles), W = 1) and two GSP-shaped single-cache traces,
with per-phase misses / first-appearance misses / clean tokens of L-LRU, OPT and R
RLT trials from kvr_sim_run_ledger, checked phase by phase against:
  * Lemma 3: L-LRU never misses an old token (misses == first misses);
  * Lemma 2: L-LRU misses <= B - L + c in every phase v >= 2;
  * Lemma 1, summed form (A23): OPT misses over phases >= 2 are at least
    sum over complete phases of max(c/2, 1) - 1, c = L-LRU's clean count;
  * Thm 3's per-phase bound from its proof: E[RLT misses in a phase with c
    clean tokens] <= c + c (H_B - H_c), c = RLT's own clean count (mean over trials).
Prints one JSON object per trace and a markdown table.

usage: python scripts/phase_ledger_sweep.py [max_log2_B=16] [rlt_trials=32] [out.json]
"""
import json
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


def H(n):
    return float(np.sum(1.0 / np.arange(1, n + 1))) if n > 0 else 0.0


def sweep(name, tr, B):
    L = int(min(tr.n_in_blocks + tr.n_out_blocks))
    t0 = time.perf_counter()
    dt = DeviceTrace(tr).with_next_use().with_phases(B)
    t_index = time.perf_counter() - t0
    sim = Simulator(1, B, pending_ring=tr.n_queries, extended_policies=True)
    pols = ([Policy(eviction=EVICT_LRU, router=ROUTE_ROUND_ROBIN),
             Policy(eviction=EVICT_OPT, router=ROUTE_ROUND_ROBIN)] +
            [Policy(eviction=EVICT_RLT, router=ROUTE_ROUND_ROBIN)] * R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res, led = sim.run_ledger(dt, np.arange(1, R + 3, dtype=np.uint64), policies_array(pols))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    assert np.all(res["status"] == 0), res["status"]
    lru, opt, rlt = led[0].astype(np.int64), led[1].astype(np.int64), led[2:].astype(np.int64)
    P = lru.shape[0]
    complete = slice(1, P - 1)          # phases 2 .. last complete one
    lemma3 = bool(np.all(lru[:, 1] == lru[:, 2]))
    slack2 = (B - L + lru[1:, 3]) - lru[1:, 1]
    lemma2 = bool(np.all(slack2 >= 0))
    c_lru = lru[complete, 3]
    lemma1_bound = float(np.sum(np.maximum(c_lru / 2.0, 1.0))) - 1.0
    lemma1 = bool(opt[1:, 1].sum() >= lemma1_bound)
    HB = H(B)
    c_r = rlt[:, :, 3]
    bound3 = c_r + c_r * (HB - np.vectorize(H)(c_r))
    mean_miss = rlt[:, 1:, 1].mean(axis=0)
    se_miss = rlt[:, 1:, 1].std(axis=0) / np.sqrt(max(1, R))
    mean_bound = bound3[:, 1:].mean(axis=0)
    row = {"trace": name, "B": B, "L": L, "queries": tr.n_queries, "blocks": tr.total_blocks,
           "phases": P, "rlt_trials": R, "index_s": t_index, "gpu_ms": ms,
           "lru_misses_per_phase": float(lru[complete, 1].mean()) if P > 2 else None,
           "lru_clean_per_phase": float(lru[complete, 3].mean()) if P > 2 else None,
           "opt_misses_per_phase": float(opt[complete, 1].mean()) if P > 2 else None,
           "rlt_misses_per_phase": float(rlt[:, complete, 1].mean()) if P > 2 else None,
           "rlt_clean_per_phase": float(rlt[:, complete, 3].mean()) if P > 2 else None,
           "lemma3_lru_no_old_misses": lemma3,
           "lemma2_lru_min_slack": int(slack2.min()) if len(slack2) else None,
           "lemma2_holds": lemma2,
           "lemma1_opt_misses": int(opt[1:, 1].sum()), "lemma1_bound": lemma1_bound,
           "lemma1_holds": lemma1,
           "thm3_rlt_phase_mean_misses_max_over_bound": float(np.max(mean_miss / np.maximum(mean_bound, 1e-9))),
           # the bound holds in expectation: per phase, the mean over R trials within 3 standard
           # errors of it
           "thm3_holds_in_mean": bool(np.all(mean_miss <= mean_bound + 3.0 * se_miss + 1e-9)),
           "thm3_max_z": float(np.max((mean_miss - mean_bound) / np.maximum(se_miss, 1e-9)))}
    print(json.dumps(row), flush=True)
    return row


rows = []
for lb in range(6, maxlog + 1):
    B = 1 << lb
    rows.append(sweep(f"ADV({B},4,8)", wl.adv(B, 4, 8, seed=0xC6), B))
for B, r in ((512, 0.3), (512, 0.9)):
    rows.append(sweep(f"GSP(128,32,{r}) W=1", wl.gsp(128, 32, r, seed=0xE0, W=1), B))

print()
print("| trace | B | phases | L-LRU misses / clean per phase | OPT misses per phase | RLT misses / clean per phase | Lemma 3 | Lemma 2 min slack | Lemma 1: OPT >= bound | Thm 3 max mean/bound (max z) | GPU ms (2 + R trials) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    f = lambda x: "-" if x is None else f"{x:.2f}"  # noqa: E731
    print(f"| {r['trace']} | {r['B']} | {r['phases']} | {f(r['lru_misses_per_phase'])} / "
          f"{f(r['lru_clean_per_phase'])} | {f(r['opt_misses_per_phase'])} | "
          f"{f(r['rlt_misses_per_phase'])} / {f(r['rlt_clean_per_phase'])} | "
          f"{'yes' if r['lemma3_lru_no_old_misses'] else 'NO'} | {r['lemma2_lru_min_slack']} | "
          f"{r['lemma1_opt_misses']} >= {r['lemma1_bound']:.0f} | "
          f"{r['thm3_rlt_phase_mean_misses_max_over_bound']:.3f} ({r['thm3_max_z']:+.1f}) | {r['gpu_ms']:.0f} |")
if out_path:
    with open(out_path, "w") as fh:
        json.dump(rows, fh, indent=1)
