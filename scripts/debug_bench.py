import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, bench, oracle
from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, Policy, policies_array
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
trs = bench.build_traces(nq)
t_of, ev, keys = bench.trial_plan(0, 6)
sim = Simulator(8, 512)
dts = [DeviceTrace(t) for t in trs]
out = sim.run(dts, keys, policies_array([Policy(eviction=int(e)) for e in ev]), trial_trace=t_of)
print("status", out.results["status"], "queries", out.results["queries"], "maxp", out.results["max_pending"])
cfg = oracle.OracleConfig(W=8, capacity_blocks=512)
for i in range(6):
    o = oracle.run(cfg, trs[t_of[i]], oracle.OraclePolicy(eviction=int(ev[i])), int(keys[i]))
    g = out.results[i]
    diff = [f for f in o.result if float(o.result[f]) != float(g[f])]
    print(i, "oracle status", o.result["status"], "q", o.result["queries"], "maxp", o.result["max_pending"], "hit", o.result["hit_tokens"], "gpu hit", g["hit_tokens"], "diff", diff)
