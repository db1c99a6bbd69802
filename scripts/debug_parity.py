import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, oracle
from paper_2601_18999_b200 import workloads as wl
from paper_2601_18999_b200 import kvr
from parity_util import run_gpu, run_oracle
W, B = int(sys.argv[1]), int(sys.argv[2]); ev = int(sys.argv[3]); router = int(sys.argv[4])
tr = wl.random_tree(300, 10 + W, max_len=min(6, B - 1), alphabet=3, max_out=1, W=W)
pols = [kvr.Policy(eviction=ev, router=router)]
cap = tr.total_blocks
out, _, _ = run_gpu(kvr, [tr], W, B, pols, [1000], (0.5, 1.0, 3.0), 256, True, cap)
o = run_oracle(oracle, tr, W, B, pols, [1000], (0.5, 1.0, 3.0), 256, True, cap)[0]
g = out.records[0]; orc = o.records
for f in ("worker", "hit_tokens", "n_victims", "victim_offset", "ttft_ms", "latency_ms", "score"):
    d = np.nonzero(g[f][:tr.n_queries] != orc[f])[0]
    print(f, "first diff", d[:5])
nv = int(o.result["evictions"])
gv = out.victims[:nv]; ov = o.victims[:nv]
d = np.nonzero(gv != ov)[0]
print("victims differ at", d[:10], "of", nv)
if len(d):
    k = d[0]
    q = int(np.searchsorted(orc["victim_offset"], k, side="right") - 1)
    print("query", q, "gpu", [hex(x) for x in gv[orc['victim_offset'][q]:orc['victim_offset'][q]+orc['n_victims'][q]]],
          "oracle", [hex(x) for x in ov[orc['victim_offset'][q]:orc['victim_offset'][q]+orc['n_victims'][q]]])
print({f: (int(out.results[0][f]) if f != 'sum_latency_ms' else float(out.results[0][f]), o.result[f]) for f in ("evictions", "decision_digest")})
