"""Queue stability of the LBGR readings at full trace length (NLMS step
mu = 0.992 (A8) vs mu = 0.008 (SPEC S:478 reading of 0.992 as a retention
factor)), and of config 3's full router grid, on one B200.

Per cell: `trials` seeded trials over the whole trace in one launch; reports the
trials that stopped at a pending-ring overflow, the largest FIFO depth, mean
latency and hit rate.  Used to choose config 3's arrival rate / ring and the
default mu.

usage: python scripts/stability_sweep.py [which=c2,c3] [trials=16] [out.json]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array  # noqa: E402

which = (sys.argv[1] if len(sys.argv) > 1 else "c2,c3").split(",")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out_path = sys.argv[3] if len(sys.argv) > 3 else None
RING = 1 << 16
rows = []


def run_cells(name, W, tr, cells, ring=RING):
    dt = DeviceTrace(tr)
    pols, keys, cell_of = [], [], []
    for c, (_, kw) in enumerate(cells):
        for t in range(K):
            pols.append(Policy(**kw))
            keys.append(1 + t)
            cell_of.append(c)
    sim = Simulator(W, 512, pending_ring=ring)
    t0 = time.time()
    out = sim.run(dt, np.array(keys, np.uint64), policies_array(pols))
    el = time.time() - t0
    res = out.results
    cell_of = np.array(cell_of)
    for c, (cname, kw) in enumerate(cells):
        r = res[cell_of == c]
        row = dict(workload=name, cell=cname, trials=int(len(r)),
                   overflow=int((r["status"] == 1).sum()), max_pending=int(r["max_pending"].max()),
                   mean_latency_ms=float((r["sum_latency_ms"] / np.maximum(r["queries"], 1)).mean()),
                   hit_rate=float(r["hit_tokens"].sum() / max(1, r["input_tokens"].sum())),
                   queries_done=float(r["queries"].mean()), wall_s=el)
        rows.append(row)
        print(json.dumps(row), flush=True)
    sim.close()


if "c2" in which:
    cells = [(f"{ev} mu={mu}", dict(eviction=e, mu=mu))
             for mu in (0.992, 0.008) for ev, e in (("RLT", 1), ("LRU", 0))]
    for util in (0.8, 0.5, 0.4):
        for r, s in zip((0.3, 0.5, 0.9), (0xC2, 0xC3, 0xC4)):
            tr = wl.gsp(125, 800, r, seed=s, W=8, util=util, lengths=(128, 256, 512, 1024, 2048))
            run_cells(f"config2 GSP r={r} util={util}", 8, tr, cells)

if "c3" in which:
    grid = ([(f"LBGR mu={mu} dt={d}", dict(router=0, mu=mu, delta_t_ms=d))
             for mu in (0.008, 0.1, 0.5, 0.992) for d in (10.0, 20.0, 40.0, 80.0)] +
            [(f"STATIC wl={a} wh={b}", dict(router=1, w_load=a, w_hit=b))
             for a in (0.25, 1.0, 4.0) for b in (0.25, 1.0, 4.0)] +
            [(f"THRESHOLD tau={tau}", dict(router=2, tau=tau)) for tau in (1.25, 1.5, 2.0, 4.0)])
    for util in (0.8, 0.5):
        tr = wl.drift(8192, 1_000_000, seed=0xC5, W=16, util=util)
        run_cells(f"config3 DRIFT util={util}", 16, tr, grid)

if out_path:
    with open(out_path, "w") as f:
        json.dump(dict(gpu=torch.cuda.get_device_name(0), trials_per_cell=K, ring=RING, rows=rows),
                  f, indent=1)
