"""One replay launch of a chosen slice of the bench workload (for ncu).

usage: python scripts/ncu_case.py [rlt|lru|mix] [queries] [trials] [batch_slots=0] [W=8]
(batch_slots > 0 runs the continuous-batching kernel, kvr_batch.cu)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import kvr  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "rlt"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
nt = int(sys.argv[3]) if len(sys.argv) > 3 else 296
beta = int(sys.argv[4]) if len(sys.argv) > 4 else 0
Wk = int(sys.argv[5]) if len(sys.argv) > 5 else 8
trs = bench.build_traces(nq)
dts = [kvr.DeviceTrace(t) for t in trs]
t_of, ev, keys = bench.trial_plan(0, nt)
if mode == "rlt":
    ev[:] = 1
elif mode == "lru":
    ev[:] = 0
sim = kvr.Simulator(Wk, 512, pending_ring=bench.RING, batch_slots=beta)
pols = kvr.policies_array([kvr.Policy(eviction=int(e)) for e in ev])
out = sim.run(dts, keys, pols, trial_trace=t_of)
torch.cuda.synchronize()
print(mode, "queries", int(out.results["queries"].sum()), "evictions",
      int(out.results["evictions"].sum()))
