import sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_18999_b200 import workloads as wl
from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, Policy, policies_array
tr = wl.random_tree(60, 5, max_len=40, alphabet=2, max_out=2, W=4, util=2.0)
for ft in (1, 2):
    sim = Simulator(4, 3 * int(tr.max_blocks), batch_slots=3, force_tier=ft, record_trials=3, latency_hist_bins=16)
    pols = [Policy(eviction=0), Policy(eviction=1), Policy(eviction=1, router=5)]
    out = sim.run(DeviceTrace(tr), np.array([1, 2, 3], np.uint64), policies_array(pols), victims_cap=3 * 4 * tr.total_blocks)
    print(ft, out.results["status"], out.results["evictions"])
