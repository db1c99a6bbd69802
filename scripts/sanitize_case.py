"""Small replays of both kernels for compute-sanitizer (memcheck / racecheck /
synccheck): the beta = 1 replay kernel (both tiers, lean and extended
instantiations, every eviction/fallback and router) and the continuous-batching
kernel (both tiers), and the split tier at W = 20.  usage: compute-sanitizer --tool X python scripts/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array  # noqa: E402

tr = wl.random_tree(60, 5, max_len=40, alphabet=2, max_out=2, W=4, util=2.0)
dt = DeviceTrace(tr)
pols = [Policy(eviction=0), Policy(eviction=1), Policy(eviction=1, rlt_fallback=1),
        Policy(eviction=1, rlt_fallback=2), Policy(eviction=1, router=1), Policy(eviction=0, router=2),
        Policy(eviction=1, router=4)]
keys = np.arange(1, len(pols) + 1, dtype=np.uint64)
B = 3 * int(tr.max_blocks)
for ft in (1, 2):
    sim = Simulator(4, B, force_tier=ft, record_trials=len(pols), latency_hist_bins=16)
    out = sim.run(dt, keys, policies_array(pols), victims_cap=len(pols) * tr.total_blocks)
    print("replay tier", ft, out.results["status"], out.results["evictions"])
    ext = [Policy(eviction=1, router=5), Policy(eviction=1, tracker_lag=1, tracker_grain=2)]
    out = sim.run(dt, keys[:2], policies_array(ext))
    print("replay ext tier", ft, out.results["status"], out.results["evictions"])
    simb = Simulator(4, B, batch_slots=3, force_tier=ft, record_trials=len(pols), latency_hist_bins=16)
    out = simb.run(dt, keys, policies_array(pols), victims_cap=len(pols) * 4 * tr.total_blocks)
    print("batch tier", ft, out.results["status"], out.results["evictions"])
# the split tier (W > 16: identities / tables in global memory, two workers per warp)
tr20 = wl.random_tree(60, 5, max_len=40, alphabet=2, max_out=2, W=20, util=2.0)
dt20 = DeviceTrace(tr20)
sim20 = Simulator(20, 3 * int(tr20.max_blocks), force_tier=3, record_trials=len(pols), latency_hist_bins=16)
out = sim20.run(dt20, keys, policies_array(pols), victims_cap=len(pols) * tr20.total_blocks)
print("replay split tier W=20", out.results["status"], out.results["evictions"])
