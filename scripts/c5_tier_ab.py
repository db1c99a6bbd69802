"""Config-5 launches (one rank's share of the fixed list, default 1/8) per W, timed with CUDA
events, under forced state tiers: quantifies the global-memory tier's cost (tier 2) against
the shared-memory tier (tier 1) at the same W.

usage: python scripts/c5_tier_ab.py [world=8] [W,...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200.kvr import DeviceTrace, Simulator  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
Ws = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(bench.C5_WS)
for L in bench.c5_plan(0, world):
    if L.W not in Ws:
        continue
    dts = [DeviceTrace(t) for t in L.traces]
    for tier in [int(t) for t in os.environ.get("KVR_AB_TIERS", "0,1,2,3").split(",")]:
        try:
            sim = Simulator(L.W, bench.B_BLOCKS, pending_ring=L.ring, force_tier=tier)
            plan = sim.plan(max(t.max_blocks for t in L.traces))
            sim.run(dts, L.keys[:4], L.policies()[:4], trial_trace=L.trial_trace[:4])
        except Exception as e:   # tier does not fit
            print(f"W={L.W} tier={tier}: {str(e)[:80]}")
            continue
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = sim.run(dts, L.keys, L.policies(), trial_trace=L.trial_trace)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        q = float(out.results["queries"].sum())
        print(f"W={L.W} tier={tier} plan={plan}: {len(L)} trials {ms:8.1f} ms  {q / ms / 1e3:6.2f} M q-r/s",
              flush=True)
