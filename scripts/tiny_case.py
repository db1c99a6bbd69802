import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2601_18999_b200 import workloads as wl
from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, Policy, policies_array
tr = wl.gsp(4, 3, 0.5, seed=1, W=2)
sim = Simulator(2, 512)
out = sim.run(DeviceTrace(tr), np.array([1], np.uint64), policies_array([Policy(eviction=0)]))
print(out.results["status"], out.results["queries"])
