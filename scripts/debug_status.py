import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, bench, oracle
from paper_2601_18999_b200.kvr import DeviceTrace, Simulator, Policy, policies_array
trs = bench.build_traces()
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
t_of, ev, keys = bench.trial_plan(0, nt)
sim = Simulator(8, 512, pending_ring=bench.RING)
dts = [DeviceTrace(t) for t in trs]
out = sim.run(dts, keys, policies_array([Policy(eviction=int(e)) for e in ev]), trial_trace=t_of)
res = out.results
bad = np.nonzero(res["status"] != 0)[0]
print("nonzero", len(bad), "status values", np.unique(res["status"][bad]))
print("by trace", np.bincount(t_of[bad], minlength=3), "by evict", np.bincount(ev[bad], minlength=2))
print("max_pending overall", res["max_pending"].max(), "median", np.median(res["max_pending"]))
for i in bad[:5]:
    print(i, t_of[i], ev[i], res["queries"][i], res["max_pending"][i])
if len(bad):
    i = int(bad[0])
    cfg = oracle.OracleConfig(W=8, capacity_blocks=512, pending_ring=bench.RING)
    t0 = time.time()
    o = oracle.run(cfg, trs[t_of[i]], oracle.OraclePolicy(eviction=int(ev[i])), int(keys[i]))
    print("oracle", o.result["status"], o.result["queries"], o.result["max_pending"], time.time() - t0)
ok = np.nonzero(res["status"] == 0)[0][:2]
for i in ok:
    cfg = oracle.OracleConfig(W=8, capacity_blocks=512, pending_ring=bench.RING)
    o = oracle.run(cfg, trs[t_of[i]], oracle.OraclePolicy(eviction=int(ev[i])), int(keys[i]))
    diff = [f for f in o.result if float(o.result[f]) != float(res[i][f])]
    print("full-trace parity trial", i, "diff fields:", diff)
