"""Kernel time per (prefix ratio, eviction) class of the config-2 bench trials: one
full wave (resident CTAs) of identical trials over the first `queries` queries.

usage: python scripts/trial_cost.py [queries]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import kvr  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
trs = bench.build_traces(nq)
dts = [kvr.DeviceTrace(t) for t in trs]
sim = kvr.Simulator(bench.W_WORKERS, bench.B_BLOCKS, pending_ring=bench.RING)
nt = 296
for ti, r in enumerate(bench.RATIOS):
    for ev, name in ((1, "RLT"), (0, "LRU")):
        keys = np.arange(nt, dtype=np.uint64) + 77
        t_of = np.full(nt, ti, dtype=np.uint32)
        pols = kvr.policies_array([kvr.Policy(eviction=ev) for _ in keys])
        sim.run(dts, keys[:8], pols[:8], trial_trace=t_of[:8])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = sim.run(dts, keys, pols, trial_trace=t_of)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        q = float(out.results["queries"].sum())
        print(f"r={r} {name}: {ms:8.1f} ms for {nt} x {nq}  -> {ms / nq * 1e3:.2f} us/query/trial, "
              f"{q / ms / 1e3:.2f} M q-r/s, evict/q {out.results['evictions'].sum() / q:.1f}", flush=True)
